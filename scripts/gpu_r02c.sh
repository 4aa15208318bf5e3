timeout 900 python -m pytest tests/test_gpu_nccl.py -q --timeout 900 -x 2>&1 | tail -15 > gpurun_out/r02_tests_c.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c.json 2> gpurun_out/r02_bench_c.err
cat gpurun_out/r02_tests_c.log; tail -3 gpurun_out/r02_bench_c.err; cat gpurun_out/r02_bench_c.json
