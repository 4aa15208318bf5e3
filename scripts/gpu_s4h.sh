mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 2>&1 | tail -5 > gpurun_out/s4h_tests.log
timeout 600 python scripts/k1_harvest_probe.py "" > gpurun_out/s4h_probe.txt 2>&1
timeout 300 python scripts/k1_clip_once.py > gpurun_out/s4h_clip.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline --no-e2e --no-k1 > gpurun_out/s4h_bench.json 2> gpurun_out/s4h_bench.err
NSCEN=128 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_thread -s 2 -c 1 \
  -o gpurun_out/s4h_k1t python scripts/k1_harvest_probe.py "" > /dev/null 2>&1
cat gpurun_out/s4h_tests.log gpurun_out/s4h_probe.txt gpurun_out/s4h_clip.txt
python -c "import json;d=json.loads(open('gpurun_out/s4h_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['kernels'])"
