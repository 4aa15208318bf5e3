"""The paper's baseline comparison and core ablation (§VI-A, §VI-H) on the
synthetic cfg2 workload: every scenario of the 4,096-scenario batch replayed
on the GPU under each selection policy (Q26); per load level
(13 rho groups) the SLO violation ratio (Eq. 2, strict) and the exact group
P95 from the all-reduced histogram merge; over all groups the effective
accuracy (Table I accuracy of the exit that served each task,
averaged over completions) and the exit-depth histogram -- both the
library's own group counters (ES_ST_ACC_BP, ES_ST_EXIT0..7), no host
reduction.  A second block splits the violations by model (host reduction of
the per-request outputs, a study, not a product number) to show WHY a policy
wins.  Prints a table (profiles/<round>_policies.txt).  Synthetic profiles:
shapes only, not the paper's numbers (its RTX 3080 profiles are unpublished)."""
import dataclasses, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import inputs, paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine

POL = {"edgeserving": 0, "all_final": 1, "all_early": 2, "ee_lqf": 3, "ee_edf": 4, "allfinal_da": 5, "ours_bs1": 6,
       "symphony": 7, "grid": 8}
GC = es.GROUP_COLS
w = inputs.workload("cfg2")
E = w.profile.E
dtr = engine.upload_traces(w.traces, "cuda")
G = inputs.n_groups("cfg2")
rho = [0.60 + 0.05 * g for g in range(G)]
cols = [0, 4, 8, 12]
lines = [f"cfg2 synthetic (4,096 scenarios x 10k requests, tau 50 ms, M=4, E=4, B 1-16); "
         f"violation % / P95 ms per rho_full; over all loads: effective accuracy (Table I, P:500-504), "
         f"mean exit index (0 = shallowest, {E - 1} = final) and the exit-depth histogram (% of completions, P:489); "
         f"every request of the finite traces completes (drain, DESIGN.md Q13): overload backlogs count in P95 and violations",
         f"{'policy':13s}" + "".join(f"   rho {rho[g]:.2f}      " for g in cols) +
         "  eff.acc  mean exit  " + " ".join(f"exit{e:d}" for e in range(E)) + "   decisions"]
per_model = {}
for name, pid in POL.items():
    cfgs = [dataclasses.replace(c, policy=pid) for c in w.cfgs]
    h = es.es_load_profile(w.profile, cfgs)
    out, counts, p95 = engine.replay_group_stats(h, dtr, G, full=True)
    torch.cuda.synchronize()
    c = counts.cpu().numpy().astype(np.float64)
    p = p95.cpu().numpy()
    tot = c.sum(axis=0)
    comp = tot[GC.index("completed")]
    hist = np.array([tot[GC.index(f"exit{e}")] for e in range(E)])
    acc = tot[GC.index("acc_bp")] / comp / 100.0
    mean_exit = float((hist * np.arange(E)).sum() / comp)
    row = f"{name:13s}"
    for g in cols:
        row += f"  {100 * c[g, GC.index('violations')] / c[g, GC.index('completed')]:6.2f}% {p[g] / 1e3:7.1f}  "
    row += f"  {acc:6.2f}%  {mean_exit:8.3f}  " + " ".join(f"{100 * x / comp:5.1f}" for x in hist)
    row += f"  {int(tot[GC.index('decisions')]):10d}"
    lines.append(row)
    if name in ("edgeserving", "ee_edf"):
        # violations and mean exit per model over the whole batch (study only)
        ex = out["exit"].cpu().numpy()
        comp_t = out["completion"].cpu().numpy().astype(np.int64)
        arr = w.traces.arrival.astype(np.int64)
        T = comp_t - arr
        off = w.traces.arr_off
        M = w.profile.M
        mid = np.repeat(np.tile(np.arange(M), w.traces.n_scen), np.diff(off.astype(np.int64)))
        tau = w.cfgs[0].tau
        per_model[name] = [(100.0 * np.mean(T[mid == m] > tau), float(np.mean(ex[mid == m])),
                            float(np.mean(T[mid == m])) / 1e3) for m in range(M)]
lines.append("")
lines.append("per model (all loads, warmup included): violation % / mean exit / mean latency ms")
lines.append(f"{'policy':13s}" + "".join(f"   model {m} (L x{2.0 ** ((m - w.profile.M + 1) / (w.profile.M - 1)):.2f})  "
                                          for m in range(w.profile.M)))
for name, v in per_model.items():
    lines.append(f"{name:13s}" + "".join(f"   {a:6.2f}% {b:5.2f} {c:7.1f}      " for a, b, c in v))
print("\n".join(lines))
