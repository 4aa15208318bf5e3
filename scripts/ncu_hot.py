"""Hot CUDA source lines (by executed instructions and stall samples) for one kernel in an ncu report."""
import subprocess, sys, os
rep, k = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
key = sys.argv[4] if len(sys.argv) > 4 else "stall"
here = os.path.dirname(os.path.abspath(__file__))
out = subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), rep, k, "400"], capture_output=True, text=True).stdout.splitlines()
print(out[0])
rows = []
for l in out[1:]:
    p = l.split()
    rows.append((p[0], float(p[2].rstrip('%')), float(p[4].rstrip('%'))))
rows.sort(key=lambda r: -(r[2] if key == "stall" else r[1]))
src = {}
d = os.path.join(os.path.dirname(here), "paper_2605_05527_b200", "csrc")
for f in os.listdir(d):
    src[f] = open(os.path.join(d, f)).read().splitlines()
acc = 0
for name, e, st in rows[:n]:
    f, ln = name.split(':') if ':' in name else (name, '0')
    text = src[f][int(ln) - 1].strip()[:90] if f in src else ''
    acc += (st if key == "stall" else e)
    print(f"{name:24s} exec {e:5.1f} stall {st:5.1f} cum {acc:5.1f} | {text}")
