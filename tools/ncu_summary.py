"""Key metrics of one kernel from an ncu report (details + raw pages)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block", "Grid Size", "Block Size"]
seen = set()
for r in csv.reader(io.StringIO(det)):
    if len(r) > 3 and r[-3] in want and r[-3] not in seen:
        seen.add(r[-3])
        print(f"{r[-3]:40s} {r[-1]:>16s} {r[-2]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in hdr:
        i = hdr.index(k)
        print(f"{k:55s} {vals[i]:>20s} {units[i]}")
stalls = []
for h, v in zip(hdr, vals):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(s for s, _ in stalls) or 1
print("stall samples:", ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:6]))
