"""Print the SASS of one ncu report in address order with per-instruction
executed counts (warp-level) and stall samples; rows above a share threshold.
usage: ncu_sass.py <rep> [min_share_pct]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, iex, iss = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
    h.index("Warp Stall Sampling (All Samples)")
data = [(r[ia], r[isrc], float(r[iex] or 0), float(r[iss] or 0)) for r in rows[2:] if len(r) >= len(h)]
te = sum(d[2] for d in data) or 1
ts = sum(d[3] for d in data) or 1
print(f"total exec {te:.3e}")
for a, s, e, st in data:
    if 100 * e / te >= thr or 100 * st / ts >= 1:
        print(f"{a} {100*e/te:5.2f}% st {100*st/ts:4.1f}%  {s}")
