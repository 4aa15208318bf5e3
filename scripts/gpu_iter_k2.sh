# K2 iteration: parity (every K2 test) + timing of the cfg3 batch per segment width
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1100 -k "k2 or golden or full_size or group or host or determinism" 2>&1 | tail -12 > gpurun_out/iter_k2_tests.log
timeout 600 python scripts/k2_mapping.py cfg3 65536 "${VARIANTS:--,ES_LPS=8,ES_LPS=32}" > gpurun_out/iter_k2_map.txt 2>&1
cat gpurun_out/iter_k2_tests.log gpurun_out/iter_k2_map.txt
