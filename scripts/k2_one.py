"""Replay a few scenarios of cfg2 (default: scenario 0, a rho=0.60 trace) with K2:
for ncu source-level stall sampling of the per-decision chain."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
ids = np.array([int(x) for x in sys.argv[1:]] or [0])
w = inputs.workload("cfg2", scen_ids=ids)
h = es.es_load_profile(w.profile, w.cfgs)
d = es.upload_traces(w.traces, "cuda:0")
out = es.alloc_replay_out(h, len(ids), w.traces.arrival.size, "cuda:0", full=False, p95=False)
for _ in range(3):
    es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
b.record(); torch.cuda.synchronize()
st = out["stats"].cpu().numpy()
print(f"K2 {a.elapsed_time(b):.3f} ms decisions {st[:,0].tolist()} ns/decision {a.elapsed_time(b)*1e6/st[:,0].max():.0f}")
