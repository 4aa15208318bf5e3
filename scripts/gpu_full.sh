# full GPU suite + smoke + bench (TAG names the outputs)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 2>&1 | tail -15 > gpurun_out/${TAG}_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_smoke.log; tail -4 gpurun_out/${TAG}_tests.log; tail -3 gpurun_out/${TAG}_bench.err
python - <<'PY'
import json, os
t = os.environ["TAG"]
d = json.loads(open(f"gpurun_out/{t}_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], d["kernels"], "e2e", d.get("e2e", {}).get("value"))
print("roof", d["roofline"]["frac"], d["roofline"].get("chain_view"))
for k in ["k1", "k1_clip", "k1_harvested"]:
    if k in d: print(k, d[k]["ms_per_launch"], d[k]["roofline"]["frac"])
print("cfg2", d.get("cfg2", {}).get("value"), "clocks", d.get("clocks"))
PY
