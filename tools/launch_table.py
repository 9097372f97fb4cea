"""Summarise an ncu --csv launch list: per kernel the launch count, average duration, share of the
summed duration and (when captured) average DRAM bytes read + written per launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, agg = None, {}
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        k = (d["Kernel Name"][:70], d.get("ID", ""))
        agg.setdefault(k, {})[d.get("Metric Name")] = float(d["Metric Value"].replace(",", ""))
per = {}
for (name, _), m in agg.items():
    e = per.setdefault(name, {"n": 0, "t": 0.0, "b": 0.0})
    e["n"] += 1
    e["t"] += m.get("gpu__time_duration.sum", 0.0)
    e["b"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(e["t"] for e in per.values()) or 1.0
for name, e in sorted(per.items(), key=lambda x: -x[1]["t"]):
    n = e["n"]
    print(f"{n:5d} launches  avg {e['t'] / n / 1e3:10.1f} us  share {100 * e['t'] / tot:5.1f}%  "
          f"dram/launch {e['b'] / n / 1e6:9.1f} MB  {name}")
