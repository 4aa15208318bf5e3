# K2 timing per prebuilt library variant: VARIANTS="pf0 pf2" bash scripts/variants_bench.sh
for v in ${VARIANTS}; do
  for rep in 1 2; do
    ES_LIB=$PWD/variants/$v.so timeout 150 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-k1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'Gdec/s %.3f'%(d['value']/1e9), 'ms/step %.3f'%d['ms_per_step'], 'k2 ms %.3f'%d['roofline']['k2_ms'])"
  done
done
