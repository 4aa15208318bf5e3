"""Is K2 bound by the longest chain?  Time K2 on (a) the full cfg2 batch,
(b) only its rho=0.60 scenarios (the longest chains), (c) one such scenario."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es

def timeit(ids):
    w = inputs.workload("cfg2", scen_ids=ids)
    h = es.es_load_profile(w.profile, w.cfgs)
    d = es.upload_traces(w.traces, "cuda:0")
    out = es.alloc_replay_out(h, len(ids), w.traces.arrival.size, "cuda:0", full=False, p95=False)
    for _ in range(3):
        es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
    b.record(); torch.cuda.synchronize()
    st = out["stats"].cpu().numpy()
    return a.elapsed_time(b) / 10, int(st[:, 0].max()), int(st[:, 0].sum())

for name, ids in [("all 4096", np.arange(4096)), ("rho0.6 only", np.arange(0, 4096, 13)),
                  ("one rho0.6", np.array([0])), ("rho1.2 only", np.arange(12, 4096, 13))]:
    ms, mx, tot = timeit(ids)
    print(f"{name:12s} K2 {ms:.3f} ms  max decisions {mx}  total {tot}  ns/decision(max chain) {ms*1e6/mx:.0f}")
