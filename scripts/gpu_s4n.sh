mkdir -p gpurun_out
R=r02 bash scripts/sanitize_all.sh > /dev/null 2>&1
R=r02 WLS="cfg1 cfg4 cfg5a cfg5b" bash scripts/bench_configs.sh > gpurun_out/cfgs_r02.txt 2>&1
cat gpurun_out/san_r02.txt | grep -E "==|SUMMARY|ok|Error|error" | head -60
cat gpurun_out/cfgs_r02.txt | cut -c1-200
