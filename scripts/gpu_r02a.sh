nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -5 > gpurun_out/r02_tests_a.log
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-k1 > gpurun_out/r02_bench_cfg3_a.json 2> gpurun_out/r02_bench_cfg3_a.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_replay -s 1 -c 1 \
  -o gpurun_out/prof_k2_cfg3_r02a python bench.py --workload cfg3 --steps 1 --warmup 1 --ncu > gpurun_out/ncu_k2cfg3.log 2>&1
cat gpurun_out/r02_tests_a.log; tail -3 gpurun_out/r02_bench_cfg3_a.err; cat gpurun_out/r02_bench_cfg3_a.json
