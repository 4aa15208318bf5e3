"""K1 stream throughput vs queue-boundary density: the same bytes as queues of
fixed depth D (D = 4096, 1024, 256) -- how much the per-boundary work costs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
prof = inputs.synth_profile(8, 5, list(range(1, 33)))
h = es.es_load_profile(prof, [inputs.SchedCfg(tau=50000, b_max=32)])
total = 1 << 29  # 2 GiB of waits
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for D in [4096, 1024, 256]:
    nq = total // D
    n = nq // 8
    q_off = torch.arange(0, n * 8 + 1, dtype=torch.int64, device="cuda") * D
    base = torch.arange(D, 0, -1, dtype=torch.int64, device="cuda") * 100000 // D  # live, non-increasing
    waits = base.to(torch.int32).repeat(n * 8)
    ms = []
    for i in range(6):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); es.es_score_candidates(h, q_off, waits); b.record(); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(np.median(ms[2:]))
    print(f"depth {D:5d}: {n} snapshots, {t:.3f} ms, {4 * total / t / 1e6:.0f} GB/s")
