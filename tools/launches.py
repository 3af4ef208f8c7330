"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", "")) / 1e3
    tot += v
    name = r[ki].replace("(anonymous namespace)::", "").replace("dfm::", "")
    print(f"{r[ii]:>4} {v:10.1f} us  {name[:110]}")
print(f"total {tot:.1f} us")
