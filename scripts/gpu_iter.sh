# quick GPU iteration: selected tests + a short cfg3 bench line (K2 only, no extras)
T=${T:-"tests/test_gpu_parity.py -k both_mappings"}
timeout 900 python -m pytest $T -x -q --timeout 600 2>&1 | tail -15 > gpurun_out/iter_tests.log
for W in ${WL:-cfg3}; do
  timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-k1 --no-e2e --no-cpu-baseline > gpurun_out/iter_bench_$W.json 2> gpurun_out/iter_bench_$W.err
done
cat gpurun_out/iter_tests.log
for W in ${WL:-cfg3}; do tail -2 gpurun_out/iter_bench_$W.err; python -c "
import json,sys; d=json.load(open('gpurun_out/iter_bench_$W.json')); r=d['roofline']
print('$W', 'value %.3e'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'k2_ms', r.get('k2_ms'), 'frac', r.get('frac'))"; done
