mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "k2 or group or host or edge or errors or golden or full_size_cfg or many_slos or segment" 2>&1 | tail -3 > gpurun_out/s4o_tests.log
cat gpurun_out/s4o_tests.log
timeout 900 python scripts/k2_variants.py default > gpurun_out/s4o_k2var.txt 2>&1
cat gpurun_out/s4o_k2var.txt
