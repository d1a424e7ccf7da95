"""Print the key metrics and the top stall reasons / source lines of one ncu report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
want = {"Duration", "DRAM Throughput", "Memory Throughput", "Achieved Active Warps Per SM",
        "Registers Per Thread", "Executed Instructions", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Issue Slots Busy", "Theoretical Active Warps per SM"}
for r in rows[1:]:
    if r[mi] in want:
        print(f"  {r[mi]} = {r[vi]} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh = rr[0]
for vals in rr[2:]:
    st = []
    for k, v in zip(hh, vals):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
    print(f"  {vals[hh.index('Kernel Name')][:50]}  stalls (warps per issue):")
    for v, k in sorted(st, reverse=True)[:7]:
        print(f"    {v:7.2f}  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
