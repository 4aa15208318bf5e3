"""Compact per-kernel register / spill report from nvcc -Xptxas -v (CPU-side check)."""
import re, subprocess, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_05527_b200 import build as b
out = []
for src in b.sources():
    if len(sys.argv) > 1 and not any(k in src for k in sys.argv[1:]):
        continue
    r = subprocess.run([b.NVCC, *b.ARCH, *b.FLAGS, "-Xptxas", "-v", "-c", src, "-o", "/dev/null"],
                       capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-3000:]); sys.exit(1)
    name = None
    for line in r.stderr.splitlines():
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            name = m.group(1)
            name = re.sub(r"_ZN2es\d+_GLOBAL__N__\w+?_\d+_(\w+?)_cu_\w+?(\d+)", r"\1:", name)
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
        if m and name:
            stack = m.group(1); spill = m.group(2)
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            print(f"{name[:70]:70s} regs {m.group(1):>4s} stack {stack} spill {spill}")
            name = None
