"""f3: the paper's sensitivity studies as sharded GPU sweeps on a synthetic
ResNet-like profile (3 models x 4 exits {layer1, layer2, layer3, final},
batch 1-10, B_max = 10): exit-point configuration (§VI-E),
SLO threshold 20-70 ms (§VI-F), model combination with equal
traffic (§VI-G).  Each point: 512 scenarios x 5,000 Poisson
requests per load level rho_full in {0.6, 0.8, 1.0, 1.2} (one group per level),
replayed by K2; violations, the exact group P95 and the mean exit (exit-depth
counters) all from the library's group merge.  Prints violation % / P95 ms.
Synthetic profile: shapes, not the paper's numbers."""
import dataclasses, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine

RHO = [0.6, 0.8, 1.0, 1.2]
PER, NREQ = 512, 5000
base = inputs.synth_profile(3, 4, list(range(1, 11)))


def rates(prof, b_max, rho, weights):
    bi = inputs.batch_index_of(prof.bs, b_max)
    w = np.asarray(weights, np.float64)
    cost = np.array([prof.lat[m, prof.E - 1, bi] / b_max for m in range(prof.M)])
    return w * (rho / float((w * cost).sum()))


def run(prof, cfg, weights, seed=11):
    n = PER * len(RHO)
    ids = np.arange(n, dtype=np.int64)
    lam = np.array([rates(prof, cfg.b_max, RHO[s // PER], weights) for s in ids])
    D = NREQ / lam.sum(axis=1)
    segs = inputs.poisson_segments(seed, ids, lam, D)
    tr = inputs._assemble(prof.M, segs, [0] * n, [s // PER for s in ids], ids)
    h = es.es_load_profile(prof, [cfg])
    dtr = engine.upload_traces(tr, "cuda")
    out, counts, p95 = engine.replay_group_stats(h, dtr, len(RHO), full=False)
    torch.cuda.synchronize()
    c = counts.cpu().numpy().astype(np.float64)
    p = p95.cpu().numpy()
    # mean exit over the post-warmup completions: the library's exit-depth counters
    GC = es.GROUP_COLS
    hist = c[:, [GC.index(f"exit{e}") for e in range(prof.E)]].sum(axis=0)
    ex = float((hist * np.arange(prof.E)).sum() / hist.sum())
    return "".join(f"  {100 * c[g, 4] / c[g, 3]:6.2f}% {p[g] / 1e3:6.1f}" for g in range(len(RHO))) + f"   {ex:5.2f}"


hdr = f"{'':22s}" + "".join(f"   rho {r:.1f}      " for r in RHO) + "  mean exit"
print("f3 sweeps, synthetic 3 models x 4 exits x batch 1-10 (B_max 10), 512 scenarios x 5k requests per rho;"
      " violation % / P95 ms; every request of the finite traces completes (drain, DESIGN.md Q13)")
print("\n# exit-point configuration (tau 50 ms, rates 3:2:1)")
print(hdr)
for name, allowed in [("layer1+final", [0, 3]), ("layer2+final", [1, 3]), ("layer3+final", [2, 3]),
                      ("all_exits", [0, 1, 2, 3])]:
    mask = np.zeros((3, 4), np.uint8)
    mask[:, allowed] = 1
    prof = dataclasses.replace(base, mask=mask)
    print(f"{name:22s}" + run(prof, inputs.SchedCfg(tau=50000, b_max=10), [3, 2, 1]))
print("\n# SLO threshold (all exits, rates 3:2:1)")
print(hdr)
for tau in [20, 30, 40, 50, 60, 70]:
    print(f"tau {tau} ms{'':14s}" + run(base, inputs.SchedCfg(tau=tau * 1000, b_max=10), [3, 2, 1]))
print("\n# model combination (tau 50 ms, equal traffic 1:1:1)")
print(hdr)
for name, rows in [("3 x light (m0)", [0, 0, 0]), ("3 x medium (m1)", [1, 1, 1]), ("3 x heavy (m2)", [2, 2, 2]),
                   ("light+medium+heavy", [0, 1, 2]), ("2 x light + heavy", [0, 0, 2]),
                   ("light + 2 x heavy", [0, 2, 2])]:
    prof = dataclasses.replace(base, lat=np.ascontiguousarray(base.lat[rows]))
    print(f"{name:22s}" + run(prof, inputs.SchedCfg(tau=50000, b_max=10), [1, 1, 1]))
