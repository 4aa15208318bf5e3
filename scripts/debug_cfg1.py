"""Debug: replay cfg1 on the GPU with a decision log and diff against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, oracle, paper_2605_05527_b200 as es
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
w = inputs.workload(name, scen_ids=[0, 1, 2] if name != "cfg1" else None, n_req=1000 if name != "cfg1" else None)
h = es.es_load_profile(w.profile, w.cfgs)
d = es.upload_traces(w.traces, "cuda:0")
cap = 2000
out = es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], full=True, dec_cap=cap)
torch.cuda.synchronize()
print("status", es.es_device_status(h))
o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap)
g = {k: v.cpu().numpy() for k, v in out.items() if hasattr(v, "cpu")}
print("gpu stats", g["stats"][:, :9].tolist())
print("orc stats", o["stats"][:, :9].tolist())
for k in ["dec_t", "dec_m", "dec_e", "dec_B", "dec_L", "dec_S"]:
    bad = np.nonzero(g[k] != o[k])[0]
    if bad.size:
        i = bad[0]
        print(k, "first diff at", i, "gpu", g[k][max(0,i-2):i+3], "orc", o[k][max(0,i-2):i+3])
        print("   t", g["dec_t"][max(0,i-2):i+3], o["dec_t"][max(0,i-2):i+3])
        break
else:
    print("decision logs equal")
