"""Key metrics of an `ncu --set full` report (one kernel launch) as text.
usage: python tools/ncu_summary_full.py report.ncu-rep [algorithmic_bytes]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
want = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Size", "Grid Size",
        "Theoretical Occupancy", "Achieved Occupancy", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "SM Frequency")
kname = None
for r in rows[1:]:
    d = dict(zip(h, r))
    kname = kname or d.get("Kernel Name")
    if d["Metric Name"] in want:
        print(f"{d['Metric Name']:36s} {d['Metric Value']} {d.get('Metric Unit', '')}")
rr = list(csv.reader(io.StringIO(raw)))
vals = dict(zip(rr[0], rr[2]))
units = dict(zip(rr[0], rr[1]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = 0.0
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    v = float(vals[k].replace(",", "")) * scale.get(units[k], 1)
    tot += v
    print(f"{k:36s} {v / 1e6:.1f} MB")
if alg:
    print(f"{'algorithmic bytes':36s} {alg / 1e6:.1f} MB  (traffic / algorithmic = {tot / alg:.3f})")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
      for k, v in vals.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not k.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()}
t = sum(st.values()) or 1.0
print("top stalls (pc samples): " + ", ".join(f"{k} {v / t * 100:.0f}%" for k, v in
                                              sorted(st.items(), key=lambda kv: -kv[1])[:6]))
print(f"kernel: {kname}")
