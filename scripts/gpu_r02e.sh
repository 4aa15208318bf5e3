mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 800 -k "thread_mapping or golden or edge or errors" 2>&1 | tail -15 > gpurun_out/r02e_tests.log
timeout 600 python scripts/k2_mapping.py cfg3 > gpurun_out/r02e_map_cfg3.txt 2>&1
timeout 600 python scripts/k2_mapping.py cfg5b > gpurun_out/r02e_map_cfg5b.txt 2>&1
timeout 600 python scripts/k2_mapping.py cfg4 > gpurun_out/r02e_map_cfg4.txt 2>&1
cat gpurun_out/r02e_tests.log gpurun_out/r02e_map_*.txt
