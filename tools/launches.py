"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum]
--csv` launch list: launches, mean time and DRAM bytes per launch, share of device time."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ii, ki, mi, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
launch = defaultdict(dict)
for r in rows[hdr + 1:]:
    launch[(r[ii], r[ki][:100])][r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for (_, k), m in launch.items():
    a = agg[k]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    mb = f" {b / c / 1e6:9.1f} MB" if b else ""
    print(f"{c:5d} {t / c / 1e3:10.1f} us {100 * t / tot:5.1f}%{mb}  {k}")
print(f"total {tot / 1e6:.3f} ms over {len(launch)} launches")
