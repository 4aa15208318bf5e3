"""K1 timing per mapping on the bench's 5-C-shaped live snapshots
(K1_BIG=1: the bench's 65,536-snapshot batch, else 4,096 snapshots)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
prof = inputs.synth_profile(8, 5, list(range(1, 33)))
cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
if os.environ.get("K1_BIG"):
    import bench
    q_off, w0, tiles = bench.k1_batch(0)
else:
    q_off, w0 = inputs.snapshots_poisson_depth(1000, np.arange(4096), 8, 4096, [4096 / 120000.0] * 8)
    tiles = 1
h = es.es_load_profile(prof, cfgs)
dq = torch.from_numpy(q_off).cuda()
dw = torch.from_numpy(w0).cuda().repeat(tiles)
nbytes = w0.nbytes * tiles
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in sys.argv[1:] or ["stream", "block", "seg"]:
    os.environ["ES_K1"] = mode
    out = es.es_score_candidates(h, dq, dw)
    ms = []
    for i in range(8):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); es.es_score_candidates(h, dq, dw, out=out); b.record(); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = np.median(ms[2:])
    print(f"{mode:7s} {t:.3f} ms  {nbytes / t / 1e6:.0f} GB/s  ({nbytes / 1e6:.0f} MB)")
