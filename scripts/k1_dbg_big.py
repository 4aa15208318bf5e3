import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch, inputs, paper_2605_05527_b200 as es, bench
prof = inputs.synth_profile(8, 5, list(range(1, 33)))
cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
h = es.es_load_profile(prof, cfgs)
for tiles in [int(x) for x in os.environ.get("TILES", "1 2 4 8 16").split()]:
    for fast in os.environ.get("FASTS", "tma regs").split():
        os.environ["ES_K1_FAST"] = fast
        q0, w0 = inputs.snapshots_poisson_depth(1000, np.arange(1024), 8, 4096, [4096 / 120000.0] * 8)
        nw = np.uint64(w0.size)
        q_off = np.concatenate([q0[:-1] + np.uint64(t) * nw for t in range(tiles)] + [q0[-1:] + np.uint64(tiles - 1) * nw])
        dq = torch.from_numpy(q_off).cuda(); dw = torch.from_numpy(w0).cuda().repeat(tiles)
        try:
            o = es.es_score_candidates(h, dq, dw); torch.cuda.synchronize()
            print(tiles, fast, "ok", dw.numel(), int(o["m"][:5].sum()), flush=True)
        except Exception as e:
            print(tiles, fast, "FAIL", repr(e)[:200], flush=True); sys.exit(1)
