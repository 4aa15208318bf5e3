"""Attribute ncu per-SASS-instruction counts to CUDA source lines using the
cubin's line table (nvdisasm -g).  usage: ncu_lines.py <rep> <kernel-substring> [top]"""
import csv, io, os, re, subprocess, sys, tempfile
from collections import defaultdict

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2605_05527_b200", "libedgeserve.so")
kf = os.environ.get("KFILTER")  # ncu -k filter when the report holds several kernels
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] +
                     (["-k", kf] if kf else []), capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = rows[0][1]
h = rows[1]
ia, isrc, iex, iss = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
    h.index("Warp Stall Sampling (All Samples)")
body = []
for r in rows[2:]:  # the first kernel's block only (a report may hold several)
    if r and r[0] in ("Kernel Name", "Address"):
        break
    body.append(r)
data = [(int(r[ia], 16), r[isrc], float(r[iex] or 0), float(r[iss] or 0)) for r in body if len(r) >= len(h)]
base = data[0][0]
# find the cubin function
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
best = None
for cb in cubins:
    d = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
    if ksub not in d:
        continue
    # split per function
    for m in re.finditer(r"\.text\.(\S+):\n(.*?)(?=\n\s*\.section|\Z)", d, re.S):
        if ksub in m.group(1):
            best = m.group(2)
            break
    if best:
        break
lines = {}
cur = None
for ln in best.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
agg_e = defaultdict(float)
agg_s = defaultdict(float)
for a, s, e, st in data:
    key = lines.get(a - base, "?")
    agg_e[key] += e
    agg_s[key] += st
te = sum(agg_e.values())
ts = sum(agg_s.values())
print(kname[:100], f"total exec {te:.3e}")
for k, v in sorted(agg_e.items(), key=lambda x: -x[1])[:top]:
    print(f"  {k:28s} exec {100*v/te:5.1f}%  stall-samples {100*agg_s[k]/ts:5.1f}%")
