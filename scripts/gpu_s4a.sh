# session-4 baseline at HEAD: smoke, GPU suite, bench line, launch list
mkdir -p gpurun_out
TAG=s4a bash scripts/gpu_full.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4a_launches.csv \
  python bench.py --steps 2 --warmup 1 --ncu > /dev/null 2>&1
echo launches rc $?
