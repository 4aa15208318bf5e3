W=${W:-cfg3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_replay -s 1 -c 1 \
  -o gpurun_out/prof_k2_${W}_${TAG:-x} python bench.py --workload $W --steps 1 --warmup 1 --ncu --no-extra > gpurun_out/ncu_k2.log 2>&1
tail -3 gpurun_out/ncu_k2.log
