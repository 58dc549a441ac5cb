"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
data = rows[hdr + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in data:
    agg[r[ki][:100]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{len(v):5d} {sum(v) / len(v) / 1e3:10.1f} us {100 * sum(v) / tot:5.1f}%  {k}")
print(f"total {tot / 1e6:.3f} ms over {len(data)} launches")
