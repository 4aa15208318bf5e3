"""K3 (per-scenario P95 + level-0 group histogram, es_scen_stats) and the group
merge on a config's bench batch, device-timed; checks the P95s against a
second run.  python scripts/k3_time.py cfg3"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
w = inputs.workload(name, scen_ids=np.arange(S))
G = inputs.n_groups(name)
h = es.es_load_profile(w.profile, w.cfgs)
d = engine.upload_traces(w.traces, "cuda:0")
out = es.alloc_replay_out(h, S, int(w.traces.arrival.size), "cuda:0", full=False, p95=True)
es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False, p95=False)
counts = torch.zeros((G, es.ES_NGSTAT), dtype=torch.uint64, device="cuda:0")
hist0 = torch.zeros((G, es.ES_HIST_BINS), dtype=torch.uint64, device="cuda:0")
for _ in range(2):
    es.es_scen_stats(h, d["arr_off"], d["arrival"], out, G, counts, hist0, d["cfg_idx"], d["group_id"])
torch.cuda.synchronize()
ms = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    es.es_scen_stats(h, d["arr_off"], d["arrival"], out, G, counts, hist0, d["cfg_idx"], d["group_id"])
    b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
byt = 4 * w.traces.arrival.size + 8 * es.ES_NSTAT * S
m = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    engine.group_merge(h, d, out, G, group=False, with_p95=True)
    b.record(); torch.cuda.synchronize(); m.append(a.elapsed_time(b))
print(f"{name} K3 {min(ms):.3f} ms = {byt / min(ms) / 1e6:.0f} GB/s ({byt / 1e6:.0f} MB); K3 + merge {min(m):.3f} ms; p95 sum {int(out['p95'].sum().item())}")
