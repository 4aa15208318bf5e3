# compute-sanitizer memcheck on small GPU parity cases (run under gpurun)
export ES_LPS=${ES_LPS:-16}
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x --timeout 500 -k "${SAN_K:-cfg1}" 2>&1 | grep -v "^=========     Host Frame" | head -40
