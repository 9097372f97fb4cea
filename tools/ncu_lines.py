"""Per-CUDA-source-line stall samples and executed instructions from an ncu --page source
--csv --print-source sass,cuda export (top N lines)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_line = cur_src = cur_file = None
agg, execs, h = {}, {}, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split('/')[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None:
        continue
    if r[0] and r[0].strip().isdigit():
        cur_line, cur_src = int(r[0]), r[1]
    try:
        s, e = float(r[4] or 0), float(r[7] or 0)
    except (ValueError, IndexError):
        continue
    k = (cur_file, cur_line, (cur_src or '').strip()[:90])
    agg[k] = agg.get(k, 0) + s
    execs[k] = execs.get(k, 0) + e
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{v / tot * 100:5.1f}% exec={execs[k]:>12.0f} {k[0]}:{k[1]} {k[2]}")
