timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_stats -s 1 -c 1 \
  -o gpurun_out/prof_k3_${TAG:-x} python bench.py --steps 1 --warmup 1 --ncu --no-extra > gpurun_out/ncu_k3.log 2>&1
tail -2 gpurun_out/ncu_k3.log
