"""Top SASS instructions (by warp stall samples) of one ncu report:
python tools/ncu_src.py REP [N] [KERNEL_SUBSTR]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kern, data, h = None, [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        kern = r[1]
        continue
    if r and r[0] == "Address":
        h = r
        continue
    if h is None or len(r) < 3 or (want and want not in (kern or "")):
        continue
    try:
        v = float(r[h.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    data.append((v, kern[:40], r[0][-5:], r[1].strip()[:90]))
tot = sum(d[0] for d in data) or 1
for i, (v, k, a, s) in enumerate(sorted(data, reverse=True)[:n]):
    print(f"{100 * v / tot:5.1f}%  {a}  {s}")
