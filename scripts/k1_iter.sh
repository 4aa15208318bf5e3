# K1 iteration: parity tests, probe timing, launch list of one probe run
timeout 300 python -m pytest tests -m gpu -q --timeout 120 -x -k "k1 or smoke or host" 2>&1 | tail -2
timeout 120 python scripts/k1_probe.py ${MODES:-stream}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/k1_probe.py stream > gpurun_out/k1_launches.csv 2>&1
python - <<'PY'
import csv
from collections import defaultdict
d = defaultdict(list)
for r in csv.reader(open('gpurun_out/k1_launches.csv')):
    if len(r) > 10 and r[0] != 'ID':
        d[r[4][:40]].append(float(r[-1]))
for k, v in d.items():
    print(f"{k:42s} n={len(v)} median {sorted(v)[len(v)//2]/1e3:.1f} us")
PY
