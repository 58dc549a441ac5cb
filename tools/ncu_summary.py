"""Print the key sections of an `ncu --page details --csv` export."""
import csv
import sys

KEEP = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
        "Scheduler Statistics", "Warp State Statistics", "Occupancy", "Launch Statistics")
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
ki = hdr.index("Kernel Name")
si, mi, ui, vi = hdr.index("Section Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), \
    hdr.index("Metric Value")
last = None
for r in rows[1:]:
    if len(r) <= vi:
        continue
    if r[ki] != last:
        print("==", r[ki][:120])
        last = r[ki]
    if r[si] in KEEP:
        print(f"  {r[si][:22]:22s} | {r[mi][:40]:40s} | {r[vi]} {r[ui]}")
