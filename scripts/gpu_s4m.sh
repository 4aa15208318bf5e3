mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "k1" 2>&1 | tail -3 > gpurun_out/s4m_tests.log
timeout 600 python scripts/k1_harvest_probe.py "" > gpurun_out/s4m_probe.txt 2>&1
NSCEN=128 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_thread -s 2 -c 1 \
  -o gpurun_out/s4m_k1t python scripts/k1_harvest_probe.py "" > /dev/null 2>&1
cat gpurun_out/s4m_tests.log gpurun_out/s4m_probe.txt
