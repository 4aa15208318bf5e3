"""Does scenario order (which warp slots the long chains land on) change K2's
time on cfg2?  Replays the same 4,096 scenarios in three orders: as generated
(rho interleaved), long chains (low rho) first, long chains last."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine

w = inputs.workload("cfg2")
h = es.es_load_profile(w.profile, w.cfgs)
M = w.profile.M
rho = 0.60 + 0.05 * (np.arange(4096) % 13)
for name, order in [("generated", np.arange(4096)), ("long_first", np.argsort(rho, kind="stable")),
                    ("long_last", np.argsort(-rho, kind="stable"))]:
    tr = inputs.workload("cfg2", scen_ids=order).traces
    d = engine.upload_traces(tr, "cuda")
    out = es.alloc_replay_out(h, 4096, tr.arrival.size, "cuda", full=False, p95=False)
    for _ in range(3):
        es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"{name:11s} K2 {np.median(ts):.3f} ms")
