"""One K1 call on the bench's clip-path batch (5-C depth at 5-B overload
rates) for ncu: python scripts/k1_clip_once.py [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
prof = inputs.synth_profile(8, 5, list(range(1, 33)))
cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
rate = inputs.rates_for_shallow_load(prof, 32, 1.5)
q_off, w0 = inputs.snapshots_poisson_depth(2000, np.arange(4096), 8, 4096, rate)
tiles = 64
nw = np.uint64(w0.size)
q = np.concatenate([q_off[:-1] + np.uint64(t) * nw for t in range(tiles)] + [q_off[-1:] + np.uint64(tiles - 1) * nw])
h = es.es_load_profile(prof, cfgs)
dq = torch.from_numpy(q).cuda(); dw = torch.from_numpy(w0).cuda().repeat(tiles)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    out = es.es_score_candidates(h, dq, dw)
torch.cuda.synchronize()
print("slow snapshots", int(((out["flags"].cpu().numpy()) & 1).size))
ms = []
for _ in range(5):
    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_.record(); es.es_score_candidates(h, dq, dw, out=out); b_.record(); torch.cuda.synchronize()
    ms.append(a_.elapsed_time(b_))
print(f"K1 clip call {min(ms):.3f} ms (L2 warm)")
