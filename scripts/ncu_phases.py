"""Per-phase warp-instructions per decision of a k2_replay ncu capture
(--import-source, -lineinfo).  python scripts/ncu_phases.py REP DECISIONS"""
import csv
import subprocess
import sys

rep, D = sys.argv[1], float(sys.argv[2])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur = None
hdr = None
out = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        out.append((cur, int(r[0]), ie, smp, r[1][:80]))
tot = sum(o[2] for o in out)
ts = sum(o[3] for o in out) or 1
print(f"total warp-inst {tot:.4e} = {tot / D:.1f} per decision")
for f, l, ie, smp, src in sorted(out, key=lambda o: -o[2])[:40]:
    print(f"{ie / D:7.1f}/dec {smp / ts * 100:5.1f}%stall {f}:{l} {src}")
