"""K2 alone on a config's bench batch under launch variants given as
comma-separated ENV=VALUE[+ENV=VALUE] items (e.g. "ES_LPS=8,ES_LPS=16"; "-" =
the library default): device time per launch (CUDA events), decisions/s, and
a bit-exact comparison of every variant's per-scenario counters with the
first's.  python scripts/k2_mapping.py cfg3 [S] [variants]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
S = int(sys.argv[2]) if len(sys.argv) > 2 else inputs.total_scenarios(name) if name != "cfg4" else 131072
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["-"]
t0 = time.time()
w = inputs.workload(name, scen_ids=np.arange(S))
print(f"{name}: {S} scenarios, {w.traces.arrival.size} requests, generated in {time.time() - t0:.1f} s", flush=True)
h = es.es_load_profile(w.profile, w.cfgs)
d = engine.upload_traces(w.traces, "cuda:0")
out = es.alloc_replay_out(h, S, int(w.traces.arrival.size), "cuda:0", full=False, p95=False)
ref = None
for mode in modes:
    for kv in mode.split("+"):
        if "=" in kv:
            k, v = kv.split("=", 1)
            os.environ[k] = v
    for _ in range(2):
        es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    st = out["stats"].cpu().numpy().copy()
    dec = int(st[:, 0].sum())
    same = "" if ref is None else f" stats == {modes[0]}: {np.array_equal(st, ref)}"
    ref = st if ref is None else ref
    for kv in mode.split("+"):
        if "=" in kv:
            os.environ.pop(kv.split("=", 1)[0], None)
    print(f"{mode:16s} K2 {min(ms):8.3f} ms  {dec / (min(ms) / 1e3):.3e} decisions/s  status max {int(st[:, 7].max())}{same}",
          flush=True)
