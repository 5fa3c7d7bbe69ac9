"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: python tools/launch_summary.py launches.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, d = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        v = float(r[h.index("Metric Value")])
        if r[h.index("Metric Unit")] in ("usecond", "us"):
            v *= 1e3
        elif r[h.index("Metric Unit")] in ("msecond", "ms"):
            v *= 1e6
        d[r[h.index("Kernel Name")][:70]].append(v)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):4d} launches  mean {sum(v)/len(v)/1e3:9.1f} us  share {sum(v)/tot*100:5.1f}%  {k}")
