"""Debug LPS-specific failures: replicate cfg1 k times (all segments active) and diff vs oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, oracle, paper_2605_05527_b200 as es
reps = int(sys.argv[1])
w = inputs.workload("cfg1")
segs = [w.traces.scenario(0)] * reps
tr = inputs._assemble(3, segs, [0] * reps, [0] * reps, np.arange(reps))
h = es.es_load_profile(w.profile, w.cfgs)
d = es.upload_traces(tr, "cuda:0")
try:
    out = es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], full=True, p95=False, dec_cap=400)
    torch.cuda.synchronize()
    o = oracle.replay_batch(w.profile, w.cfgs, tr, dec_cap=400)
    g = out["stats"].cpu().numpy()
    print("reps", reps, "equal" if np.array_equal(g, o["stats"]) else ("DIFF", g[:, :9].tolist(), o["stats"][0, :9].tolist()))
except Exception as e:
    print("reps", reps, "ERROR", str(e)[:200])
print("devstatus", es.es_device_status(h))
