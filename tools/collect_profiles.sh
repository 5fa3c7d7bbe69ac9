#!/bin/bash
# Turn the round-end evidence in gpurun_out/ (tools/round_evidence.sh on the B200) into profiles/r02_*.
# usage: bash tools/collect_profiles.sh [round-tag]
r=${1:-r02}; o=gpurun_out/${r}e; p=profiles
mkdir -p $p
last_json() { python -c "import json,sys; print(json.dumps(json.loads([l for l in open('$1') if l.startswith('{')][-1]), indent=1))"; }
last_json ${o}_bench.json > $p/${r}_bench.json
last_json ${o}_bench_ref.json > $p/${r}_bench_reference.json
cp ${o}_smi.txt $p/${r}_gpu.txt
tail -4 ${o}_pytest.log > $p/${r}_pytest_gpu_tail.txt
cp ${o}_smoke.log $p/${r}_smoke.txt
cp ${o}_bench_launches.csv $p/${r}_bench_launches.csv
{ echo "ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py --steps 3 --warmup 3 (cold-cache, serialised launches)";
  python tools/launch_summary.py ${o}_bench_launches.csv; } > $p/${r}_bench_launch_summary.txt
python tools/ncu_summary.py ${o}_thc_fused.ncu-rep > $p/${r}_thc_fused_ncu_full.txt 2>&1
FN=ILi10ELb1E python tools/ncu_lines.py ${o}_thc_fused.ncu-rep ${EVIDENCE_LIB:-paper_2407_01378_b200/libgradcomp_b200.so} \
  paper_2407_01378_b200/csrc/gc_thc_fused.cu thc_fused > $p/${r}_thc_fused_lines.txt 2>&1
python tools/ncu_summary.py ${o}_psgd_tma.ncu-rep > $p/${r}_psgd_tma_ncu_full.txt 2>&1
python tools/ncu_summary.py ${o}_thc_rank.ncu-rep > $p/${r}_thc_rank_ncu_full.txt 2>&1
python tools/ncu_summary.py ${o}_mtp_umma.ncu-rep > $p/${r}_mtp_umma_ncu_full.txt 2>&1
python tools/ncu_summary.py ${o}_psgd_async.ncu-rep > $p/${r}_psgd_async_ncu_full.txt 2>&1
cp ${o}_umma_rate.jsonl $p/${r}_umma_rate.jsonl
cp ${o}_unaligned_stream.jsonl $p/${r}_unaligned_stream.jsonl
grep -v NCCL ${o}_rank.jsonl > $p/${r}_rank_350m.jsonl
for s in thc psgd psgd_gpt2 psgd_gpt2_dist fp16; do
  { echo "ncu launch list of one per-rank round at d = 350M (tools/time_rank.py --scheme $s): cold-cache, serialised";
    python tools/launch_summary.py ${o}_rank_${s}_launches.csv; } > $p/${r}_rank_${s}_launch_summary.txt
done
cp ${o}_sweep_synthetic.jsonl $p/${r}_sweep_synthetic.jsonl
cp ${o}_sweep_dims.jsonl $p/${r}_sweep_dims.jsonl
cp ${o}_nmse_sweep.txt $p/${r}_nmse_sweep.txt
cp ${o}_ref_tests_seam.txt $p/${r}_reference_tests_through_b200_seam.txt
cp ${o}_ref_tests_core.txt $p/${r}_reference_tests_through_ctypes_core.txt
for t in memcheck racecheck synccheck; do cp ${o}_san_${t}.txt $p/${r}_sanitizer_${t}.txt; done
# roofline.traffic for the bench line: DRAM bytes of the captured thc_fused launch
python - <<'PY'
import csv, io, json, subprocess
rep = "gpurun_out/r02e_thc_fused.ncu-rep"
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
def get(k):
    x = float(v[h.index(k)].replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[h.index(k)], 1)
tr = json.load(open("profiles/traffic.json"))
key = "thc_fused_kernel:n=8:d=25557032:q=4:b=8:B=1024"
tr[key] = int(get("dram__bytes_read.sum") + get("dram__bytes_write.sum"))
sms, ghz = 148, 1.965
tr["issue:" + key] = {"warp_instructions_per_launch": int(get("smsp__inst_executed.sum")),
                      "peak_warp_inst_per_s": sms * 4 * ghz * 1e9,
                      "peak_source": "4 schedulers x 148 SMs x 1 warp-instruction / cycle at 1965 MHz",
                      "issue_active_frac_ncu": get("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100}
tr["_source"] = ("ncu --set full --clock-control none, one launch of thc_fused_kernel<10,1> at cfg2 "
                 "(profiles/r02_thc_fused_ncu_full.txt): dram__bytes_read.sum + dram__bytes_write.sum, smsp__inst_executed.sum")
json.dump(tr, open("profiles/traffic.json", "w"), indent=1)
PY
ls -la $p | tail -40
