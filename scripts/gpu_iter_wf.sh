mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1100 -k "k2 or golden or full_size" 2>&1 | tail -5 > gpurun_out/iter_wf_tests.log
for lib in libedgeserve libes_wf1 libes_wf4; do
  echo "== $lib" >> gpurun_out/iter_wf_map.txt
  ES_LIB=$PWD/paper_2605_05527_b200/$lib.so timeout 600 python scripts/k2_mapping.py cfg3 65536 "ES_LPS=8,ES_LPS=16" 2>&1 | grep K2 >> gpurun_out/iter_wf_map.txt
done
cat gpurun_out/iter_wf_tests.log gpurun_out/iter_wf_map.txt
