"""Small invocations of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck): K-tables, K2 at every segment width (8 / 16
/ 32 lanes) with the decision log, the policy and GRID instantiations, K3 +
the group merge levels, K1 warp-segment mapping and the K1 TMA-ring stream
(5-C-shaped deep snapshots) with its clip path.  Each case is checked against
the oracle so a sanitizer run is also a parity run.  Usage:
    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py [case ...]"""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import inputs
import oracle
import paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine

DEV = "cuda:0"


def k2(name, ids, n_req, lps=None, policy=None):
    if lps:
        os.environ["ES_LPS"] = str(lps)
    w = inputs.workload(name, scen_ids=np.asarray(ids), n_req=n_req)
    cfgs = w.cfgs if policy is None else [dataclasses.replace(c, policy=policy) for c in w.cfgs]
    h = es.es_load_profile(w.profile, cfgs)
    d = es.upload_traces(w.traces, DEV)
    out = es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], full=True, dec_cap=64)
    G = int(w.traces.group_id.max()) + 1
    counts, p95 = engine.group_merge(h, d, out, G, group=False, with_p95=True)
    torch.cuda.synchronize()
    os.environ.pop("ES_LPS", None)
    ref = oracle.replay_batch(w.profile, cfgs, w.traces, full=True, dec_cap=64)
    assert np.array_equal(out["stats"].cpu().numpy(), ref["stats"]), name
    assert np.array_equal(out["p95"].cpu().numpy(), ref["p95"]), name
    assert np.array_equal(out["dec_m"].cpu().numpy(), ref["dec_m"]), name
    return f"{name} ids={list(ids)[:4]} n_req={n_req} lps={lps} policy={policy}: ok"


def k1_segment():
    prof = inputs.synth_profile(4, 4, [1, 2, 4, 8, 16])
    cfgs = [inputs.SchedCfg(tau=50000, b_max=10), inputs.SchedCfg(tau=20000, b_max=7)]
    q_off, w = inputs.snapshots_uniform(3, 600, 4, 10, 150000)
    ci = (np.arange(600) % 2).astype(np.uint16)
    h = es.es_load_profile(prof, cfgs)
    os.environ["ES_K1"] = "seg"
    g = es.es_score_candidates(h, torch.from_numpy(q_off).to(DEV), torch.from_numpy(w).to(DEV),
                               torch.from_numpy(ci).to(DEV))
    torch.cuda.synchronize()
    os.environ.pop("ES_K1")
    r = oracle.decide_batch(prof, cfgs, q_off, w, ci)
    for k in ["m", "e", "B", "L", "S", "flags"]:
        assert np.array_equal(g[k].cpu().numpy(), r[k]), k
    return "k1 warp-segment: ok"


def k1_thread():
    """Thread-per-snapshot mapping: one SLO, regions over several shared-memory
    chunks, a misaligned waits view, planted inversions (per-lane redo), a few
    clip-path snapshots (handed to the warp segments), mixed SLOs in one warp."""
    M = 8
    prof = inputs.synth_profile(M, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32), inputs.SchedCfg(tau=90000, b_max=20)]
    n = 32 * 9 + 5
    q_off, w = inputs.snapshots_uniform(11, n, M, 60, 60000)
    w = w.copy()
    for s in (7, 100, 200):  # clip path
        lo = int(q_off[s * M])
        if int(q_off[s * M + 1]) > lo:
            w[lo] = 200000
    for s in (40, 150):  # inversions inside a queue
        lo, hi = int(q_off[s * M + 2]), int(q_off[s * M + 3])
        if hi - lo >= 3:
            w[lo + 2] = w[lo + 1] + 1
    ci = np.zeros(n, np.uint16)
    ci[64 + 3] = 1
    h = es.es_load_profile(prof, cfgs)
    buf = np.zeros(w.size + 1, np.uint32)
    buf[1:] = w
    dw = torch.from_numpy(buf).to(DEV)[1:]
    os.environ["ES_K1"] = "thread"
    g = es.es_score_candidates(h, torch.from_numpy(q_off).to(DEV), dw, torch.from_numpy(ci).to(DEV))
    torch.cuda.synchronize()
    os.environ.pop("ES_K1")
    r = oracle.decide_batch(prof, cfgs, q_off, w, ci)
    for k in ["m", "e", "B", "L", "S", "flags"]:
        assert np.array_equal(g[k].cpu().numpy(), r[k]), k
    return "k1 thread per snapshot (balanced pass, chunks, misaligned, inversions, clip list, mixed SLOs): ok"


def k1_stream(shallow):
    prof = inputs.synth_profile(8, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
    rate = inputs.rates_for_shallow_load(prof, 32, 1.5) if shallow else [2048 / 120000.0] * 8
    q_off, w = inputs.snapshots_poisson_depth(5, np.arange(40), 8, 2048, rate)
    h = es.es_load_profile(prof, cfgs)
    os.environ["ES_K1"] = "stream"
    g = es.es_score_candidates(h, torch.from_numpy(q_off).to(DEV), torch.from_numpy(w).to(DEV))
    torch.cuda.synchronize()
    os.environ.pop("ES_K1")
    r = oracle.decide_batch(prof, cfgs, q_off, w)
    for k in ["m", "e", "B", "L", "S", "flags"]:
        assert np.array_equal(g[k].cpu().numpy(), r[k]), k
    return f"k1 TMA stream ({'clip path' if shallow else 'all live'}): ok"


CASES = {
    "cfg1": lambda: k2("cfg1", [0], 1000),
    "cfg2_l8": lambda: k2("cfg2", [1, 2, 3, 4, 5, 6, 7, 8], 1500, lps=8),
    "cfg2_l16": lambda: k2("cfg2", [1, 2, 3, 4, 5, 6, 7, 8], 1500, lps=16),
    "cfg3_l32": lambda: k2("cfg3", [2, 11, 40, 77], 1200, lps=32),
    "cfg3_l16": lambda: k2("cfg3", [2, 11, 40, 77], 1200, lps=16),
    "cfg2_edf": lambda: k2("cfg2", [1, 2, 3, 4], 1200, policy=4),
    "cfg2_symphony": lambda: k2("cfg2", [1, 2, 3, 4], 1200, policy=7),
    "cfg2_grid": lambda: k2("cfg2", [1, 2], 600, policy=8),
    "k1_seg": k1_segment,
    "k1_thread": k1_thread,
    "k1_stream": lambda: k1_stream(False),
    "k1_clip": lambda: k1_stream(True),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        print(CASES[n](), flush=True)
