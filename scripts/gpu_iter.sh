# quick iteration: parity (gpu tests), bench K2 timing per LPS, ncu of K2 at the default LPS
timeout 400 python -m pytest tests -m gpu -q --timeout 120 -x 2>&1 | tail -3 | tee gpurun_out/tests.log
for L in ${LPS_LIST:-8 16}; do ES_LPS=$L timeout 150 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LPS',$L, 'Gdec/s %.3f'%(d['value']/1e9), 'ms/step %.3f'%d['ms_per_step'], 'k2 ms %.3f'%d['roofline']['k2_ms'])"; done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_replay -s 1 -c 1 -o gpurun_out/prof_k2_$NCU python bench.py --steps 1 --warmup 1 --ncu > gpurun_out/ncu_$NCU.log 2>&1; tail -1 gpurun_out/ncu_$NCU.log
fi
