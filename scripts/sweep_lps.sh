# GPU sweep: parity at each lanes-per-scenario setting, then the bench K2 time
timeout 200 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
for L in ${LPS_LIST:-8 16 32}; do echo "== LPS $L"; ES_LPS=$L ES_K1_LPS=$L timeout 400 python -m pytest tests -m gpu -q --timeout 120 -x 2>&1 | tail -3; done
for L in ${LPS_LIST:-8 16 32}; do ES_LPS=$L timeout 150 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LPS',$L, 'Gdec/s %.3f'%(d['value']/1e9), 'ms/step %.3f'%d['ms_per_step'], 'k2 ms %.3f'%d['roofline']['k2_ms'])"; done
