"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count/avg/share."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
h, agg = None, {}
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg.setdefault(d["Kernel Name"][:70], []).append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):5d} launches  avg {sum(v)/len(v)/1e3:10.1f} us  share {100*sum(v)/tot:5.1f}%  {k}")
