mkdir -p gpurun_out
ES_K2=thread timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "k2 or group or host or edge or errors or golden or full_size_cfg" 2>&1 | tail -15 > gpurun_out/s4j_tests.log
cat gpurun_out/s4j_tests.log
timeout 900 python scripts/k2_variants.py default "default+ES_K2=seg" > gpurun_out/s4j_k2var.txt 2>&1
cat gpurun_out/s4j_k2var.txt
