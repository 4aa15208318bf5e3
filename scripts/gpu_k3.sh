timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "group or p95 or full_size or k2_parity or edge or golden or host" 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-k1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k3.json 2> gpurun_out/k3.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/k3.json')); print(d['kernels'], d['ms_per_step'], '%.3e'%d['value'])"
