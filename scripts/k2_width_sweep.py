"""K2 time per segment width (ES_LPS) on each config's bench batch (1 GPU).
python scripts/k2_width_sweep.py cfg2:8,16 cfg3:16,32 ..."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_05527_b200 as es  # noqa: E402

for arg in sys.argv[1:]:
    name, widths = arg.split(":")
    t0 = time.time()
    w, S = bench.rank_workload(name, 0, int(os.environ.get("SCEN", "0")) or None)
    h = es.es_load_profile(w.profile, w.cfgs, device=0)
    d = es.upload_traces(w.traces, "cuda:0")
    gen = time.time() - t0
    out = None
    for lps in widths.split(","):
        os.environ["ES_LPS"] = lps
        ts = []
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out,
                                      full=False, p95=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        dec = float(out["stats"][:, 0].sum().item())
        print(f"{name} S={S} lps={lps} K2 ms {min(ts[1:]):.2f} (median {np.median(ts[1:]):.2f}) "
              f"decisions/s {dec / min(ts[1:]) * 1e3:.3e} (gen {gen:.0f}s)", flush=True)
