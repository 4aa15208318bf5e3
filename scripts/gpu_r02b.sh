timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -15 > gpurun_out/r02_tests_b.log
cat gpurun_out/r02_tests_b.log
