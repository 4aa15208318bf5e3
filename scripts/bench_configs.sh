# bench lines for the other BASELINE configs (per-GPU shards, K2+K3+group merge per step)
R=${R:-r01}
for W in ${WLS:-cfg3 cfg4 cfg5b cfg5a cfg1}; do
  timeout 900 python bench.py --workload $W --steps ${STEPS:-5} --warmup 3 --no-e2e --no-k1 \
    > gpurun_out/bench_${R}_$W.json 2> gpurun_out/bench_${R}_$W.err
  echo "$W rc=$? $(tail -c 300 gpurun_out/bench_${R}_$W.json)"
  tail -1 gpurun_out/bench_${R}_$W.err
done
