"""Per-source-line executed-instruction and stall-sample shares of an ncu report.
usage: python tools/ncu_lines.py report.ncu-rep object.o source.cu [kernel-substring]"""
import csv, collections, io, os, re, subprocess, sys, tempfile
rep, obj, srcf = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = rows[0][1] if len(rows[0]) > 1 else ""
h = rows[1]; ix = h.index("Instructions Executed"); isamp = h.index("Warp Stall Sampling (All Samples)"); isrc = h.index("Source")
data = [(int(r[0], 16), float(r[ix] or 0), float(r[isamp] or 0)) for r in rows[2:] if len(r) > ix and r[0].startswith("0x")]
base = min(a for a, _, _ in data)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
want = sys.argv[4] if len(sys.argv) > 4 else None
dis = ""
for cubin in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):   # a .so holds one per .cu
    text = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
    if want is None or want in text:
        dis = text
        break
# map function name -> address->line
lm = {}; cur = None; infn = False
for line in dis.split("\n"):
    if line.startswith(".text."):   # FN (env) narrows to one template instance's mangled name
        infn = (want is None or want in line) and os.environ.get("FN", "") in line
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', line) if "//##" in line else None
    if m:   # (file, line): the source file asked for and the headers it inlines
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', line)
    if m2 and cur and infn: lm[int(m2.group(1), 16)] = cur
ci = collections.Counter(); cs = collections.Counter()
for a, c, s in data:
    l = lm.get(a - base, ("?", -1)); ci[l] += c; cs[l] += s
ti, ts = sum(ci.values()), sum(cs.values())
srcdir = os.path.dirname(os.path.abspath(srcf))
cache = {}
def text(f, l):
    if f not in cache:
        path = os.path.join(srcdir, f)
        cache[f] = open(path).read().split("\n") if os.path.exists(path) else []
    lines = cache[f]
    return lines[l - 1].strip()[:80] if 0 < l <= len(lines) else "?"
print(f"{kname[:80]}: {ti:.3g} warp-instr, {ts:.3g} samples")
for (f, l), c in ci.most_common(int(os.environ.get("TOP", 30))):
    print(f"{f[:18]:18s}:{l:4d} inst {c/ti*100:5.1f}%  stall {cs[(f, l)]/ts*100:5.1f}%  {text(f, l)}")
