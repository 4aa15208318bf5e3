"""The paper's baseline comparison and core ablation (§VI-A, §VI-H) on the
synthetic cfg2 workload: every scenario of the 4,096-scenario batch replayed
on the GPU under each selection policy (Q26); per load level
(13 rho groups) the SLO violation ratio (Eq. 2, strict) and the exact group
P95 from the all-reduced histogram merge; overall mean exit depth.  Prints a
table (profiles/<round>_policies.txt).  Synthetic profiles: shapes only, not
the paper's numbers (its RTX 3080 profiles are unpublished)."""
import dataclasses, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine

POL = {"edgeserving": 0, "all_final": 1, "all_early": 2, "ee_lqf": 3, "ee_edf": 4, "allfinal_da": 5, "ours_bs1": 6,
       "symphony": 7, "grid": 8}
w = inputs.workload("cfg2")
dtr = engine.upload_traces(w.traces, "cuda")
G = inputs.n_groups("cfg2")
rho = [0.60 + 0.05 * g for g in range(G)]
cols = [0, 4, 8, 12]
lines = [f"cfg2 synthetic (4,096 scenarios x 10k requests, tau 50 ms, M=4, E=4, B 1-16); "
         f"violation % / P95 ms per rho_full; mean exit index (0 = shallowest, {w.profile.E - 1} = final)",
         f"{'policy':13s}" + "".join(f"   rho {rho[g]:.2f}      " for g in cols) + "  mean exit  decisions"]
for name, pid in POL.items():
    cfgs = [dataclasses.replace(c, policy=pid) for c in w.cfgs]
    h = es.es_load_profile(w.profile, cfgs)
    out, counts, p95 = engine.replay_group_stats(h, dtr, G, full=True)
    torch.cuda.synchronize()
    c = counts.cpu().numpy().astype(np.float64)
    p = p95.cpu().numpy()
    ex = out["exit"].to(torch.float64).mean().item()
    row = f"{name:13s}"
    for g in cols:
        row += f"  {100 * c[g, 4] / c[g, 3]:6.2f}% {p[g] / 1e3:7.1f}  "
    row += f"  {ex:8.3f}  {int(c[:, 0].sum()):10d}"
    lines.append(row)
print("\n".join(lines))
