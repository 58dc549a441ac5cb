"""Summarise an ncu SASS source page export: instruction mix and hot lines.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv; python tools/sass_hot.py X.csv [min_exec]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ie]), r[src].strip(), int(r[st] or 0), r[0]))
    except ValueError:
        continue
tot = sum(d[0] for d in data)
print("warp instructions", tot, "stall samples", sum(d[2] for d in data))
mix = Counter()
for n, s, _, _ in data:
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    mix[op.split(".")[0]] += n
print(", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in mix.most_common(14)))
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
for n, s, stall, addr in data:
    if n >= lim:
        print(addr[-5:], n, stall, s)
