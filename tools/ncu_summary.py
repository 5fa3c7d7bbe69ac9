"""Summarise an ncu report: key metrics, stall reasons, opcode mix and hottest SASS lines.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv, collections, subprocess, sys, io

rep = sys.argv[1]
def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
hdr, units = raw[0], raw[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
        # tensor pipe (tcgen05) and TMA: the PowerSGD GEMMs' utilisation counters
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"]
for row in raw[2:]:
    name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print("==", name[:90])
    for k in keys:
        if k in hdr:
            print(f"  {k:70s} {row[hdr.index(k)]:>16s} {units[hdr.index(k)]}")
    stalls = [(h, row[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    stalls = sorted(((float(v.replace(",", "")), h) for h, v in stalls if v), reverse=True)[:8]
    print("  stalls/issue:", ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={v:.2f}" for v, h in stalls))

src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
if len(src) > 2:
    h = src[1]
    ix, isamp, isrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    agg = collections.Counter(); samp = collections.Counter(); tot = tots = 0; lines = []
    for r in src[2:]:
        if len(r) <= ix: continue
        op = r[isrc].strip().split()
        if not op: continue
        o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
        try: c = float(r[ix] or 0); s = float(r[isamp] or 0)
        except ValueError: continue
        agg[o] += c; samp[o] += s; tot += c; tots += s; lines.append((s, r[0], r[isrc]))
    print(f"  warp-instructions executed {tot:.3g}, stall samples {tots:.3g}")
    print("  opcode mix: " + ", ".join(f"{o} {c/tot*100:.1f}%" for o, c in agg.most_common(16)))
    print("  hottest:")
    for s, a, t in sorted(lines, reverse=True)[:12]:
        print(f"    {s/tots*100:5.1f}%  {t.strip()[:80]}")
