# K1 TMA-ring iteration: K1 parity tests, probe timing per consumer-warp count, launch list
for NW in ${NWS:-16 24 32}; do ES_K1_NW=$NW timeout 300 python -m pytest tests -m gpu -q --timeout 120 -x -k "k1" 2>&1 | tail -1 | sed "s/^/NW=$NW /"; done
for NW in ${NWS:-16 24 32}; do ES_K1_NW=$NW timeout 120 python scripts/k1_probe.py stream | sed "s/^/NW=$NW /"; done
ES_K1_FAST=regs timeout 120 python scripts/k1_probe.py stream | sed "s/^/regs /"
ES_K1_NW=${NCU_NW:-32} timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv python scripts/k1_probe.py stream > gpurun_out/k1_launches.csv 2>&1
python - <<'PY'
import csv
from collections import defaultdict
d = defaultdict(list)
for r in csv.reader(open('gpurun_out/k1_launches.csv')):
    if len(r) > 10 and r[0] != 'ID' and r[-3] == 'gpu__time_duration.sum':
        d[r[4][:40]].append(float(r[-1]))
for k, v in d.items():
    print(f"{k:42s} n={len(v)} median {sorted(v)[len(v)//2]/1e3:.1f} us")
PY
