mkdir -p gpurun_out
ES_K2=thread timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "k2 or group or host or edge or errors or golden or full_size_cfg" 2>&1 | tail -3 > gpurun_out/s4k_tests.log
cat gpurun_out/s4k_tests.log
timeout 900 python scripts/k2_variants.py default > gpurun_out/s4k_k2var.txt 2>&1
cat gpurun_out/s4k_k2var.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_thread -c 1 \
  -o gpurun_out/s4k_k2t python scripts/k2_variants.py default > /dev/null 2>&1
