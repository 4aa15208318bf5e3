"""Pins of the oracle's whole-trace replay (online loop P:161-167, exclusive
time-division execution P:152-153) and statistics (Eq. 1-2, P95).

Pinned against closed forms (single request, M/D/1 Pollaczek-Khinchine mean
wait), the SPEC examples, structural invariants that any correct schedule of
the paper's system satisfies, an independent mini-executor and an exhaustive
action-tree search on toy traces (oracle/bruteforce.py).
"""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle
from oracle import bruteforce as bf

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def traces_from(per_scen, cfg_idx=None):
    """per_scen: list of per-model lists of arrival times."""
    M = len(per_scen[0])
    segs = [[np.asarray(q, np.uint32) for q in sc] for sc in per_scen]
    n = len(per_scen)
    return inputs._assemble(M, segs, cfg_idx if cfg_idx is not None else [0] * n, [0] * n,
                            np.arange(n))


def prof1(L, E=1):
    lat = np.asarray(L, np.uint32).reshape(1, E, -1)
    return inputs.Profile(M=1, E=E, bs=np.arange(1, lat.shape[2] + 1, dtype=np.int32), lat=lat,
                          mask=np.ones((1, E), np.uint8))


def test_single_request_golden():
    """one arrival at t=0 with L=28000 completes at 28000, T=28000."""
    ex = GOLD["run"][0]
    prof = prof1([ex["L_us"]])
    tr = traces_from([[[ex["arrival_us"]]]])
    o = oracle.replay_batch(prof, [inputs.SchedCfg(tau=50000, b_max=1, warmup=0)], tr)
    assert int(o["completion"][0]) == ex["completion_us"]
    assert int(o["lat"][0]) == ex["completion_us"] - ex["arrival_us"]
    assert int(o["p95"][0]) == 28000 and int(o["stats"][0, 0]) == 1


def test_same_instant_arrivals_do_not_overlap():
    """two arrivals at t=0 to two models: the second batch starts when the
    first completes (time-division exclusivity)."""
    prof = inputs.synth_profile(2, 2, [1])
    tr = traces_from([[[0], [0]]])
    o = oracle.replay_batch(prof, [inputs.SchedCfg(tau=50000, b_max=1, warmup=0)], tr, dec_cap=4)
    L0, L1 = int(o["dec_L"][0]), int(o["dec_L"][1])
    assert int(o["dec_t"][0]) == 0 and int(o["dec_t"][1]) == L0
    assert sorted(o["completion"].tolist()) == [L0, L0 + L1]


def test_md1_pollaczek_khinchine():
    """M=1, E=1, bs={1}, rho=0.5, D=10 ms: mean wait rho D / (2 (1 - rho))
    = 5000 us (M/D/1), within statistical error."""
    D = 10000
    prof = prof1([D])
    lam = 0.5 / D
    n_req = 150000  # 3e9 us of trace: stays inside u32 time (Q19)
    segs = inputs.poisson_segments(11, [0], np.array([[lam]]), np.array([n_req / lam]))
    tr = inputs._assemble(1, segs, [0], [0], [0])
    cfg = [inputs.SchedCfg(tau=1 << 20, b_max=1, warmup=1000)]
    o = oracle.replay_batch(prof, cfg, tr)
    st = o["stats"][0]
    mean_wait = st[8] / st[3] - D  # T = w + t (Eq. 1), t = D
    assert abs(mean_wait - 5000.0) < 250.0, mean_wait


def _check_invariants(prof, cfgs, tr, o, dec_cap):
    M = prof.M
    for s in range(tr.n_scen):
        c = cfgs[int(tr.cfg_idx[s])]
        arr = tr.scenario(s)
        lo = int(tr.arr_off[s * M])
        hi = int(tr.arr_off[s * M + M])
        comp = o["completion"][lo:hi]
        lat = o["lat"][lo:hi]
        ex = o["exit"][lo:hi]
        nd = int(o["stats"][s, 0])
        assert nd <= dec_cap
        d = slice(s * dec_cap, s * dec_cap + nd)
        t, L, m_, e_, B_ = (o["dec_t"][d].astype(np.int64), o["dec_L"][d].astype(np.int64),
                            o["dec_m"][d], o["dec_e"][d], o["dec_B"][d].astype(np.int64))
        # conservation: every request served exactly once
        assert int(B_.sum()) == hi - lo
        # exclusivity + work conservation: a batch starts exactly at the previous
        # completion unless every queue was empty, then at the next arrival
        allarr = np.sort(np.concatenate(arr).astype(np.int64))
        assert t[0] == allarr[0]
        for k in range(1, nd):
            assert t[k] >= t[k - 1] + L[k - 1]
            if t[k] > t[k - 1] + L[k - 1]:
                # idle gap: nothing pending, next arrival lands exactly at t[k]
                served = int(B_[:k].sum())
                arrived = int(np.searchsorted(allarr, t[k - 1] + L[k - 1], side="right"))
                assert arrived == served
                assert t[k] in set(allarr.tolist())
        # per-request: completion = t + L of its batch, FIFO within each queue,
        # T = completion - arrival (Eq. 1), exits from the decision
        head = [0] * M
        off = [int(tr.arr_off[s * M + m]) - lo for m in range(M)]
        seq = 0
        for k in range(nd):
            m = int(m_[k])
            for j in range(int(B_[k])):
                i = off[m] + head[m] + j
                assert comp[i] == t[k] + L[k]
                assert ex[i] == e_[k]
                assert arr[m][head[m] + j] <= t[k]  # causality
                assert lat[seq] == comp[i] - arr[m][head[m] + j]
                if o["dec_f"][s * dec_cap + k]:
                    assert lat[seq] <= c.tau  # Eq. 6 guarantee
                seq += 1
            head[m] += int(B_[k])
        # statistics (Eq. 2 strict, Q14 warmup, Q15 nearest rank)
        post = lat[c.warmup:]
        assert int(o["stats"][s, 3]) == post.size
        assert int(o["stats"][s, 4]) == int((post > c.tau).sum())
        if post.size:
            k = math.ceil(0.95 * post.size)
            assert int(o["p95"][s]) == int(np.sort(post)[k - 1])


@pytest.mark.parametrize("name,ids", [("cfg1", [0]), ("cfg2", [0, 5, 12]), ("cfg3", [0, 4, 8, 30])])
def test_replay_invariants(name, ids):
    w = inputs.workload(name, scen_ids=ids, n_req=2000 if name != "cfg1" else None)
    cap = 4096
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap)
    _check_invariants(w.profile, w.cfgs, w.traces, o, cap)
    o2 = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap, nthreads=3)
    for k in o:  # determinism, independent of the thread split
        assert np.array_equal(o[k], o2[k]), k


def test_decisions_match_snapshot_decide():
    """Each replay decision equals decide() on the harvested queue snapshot."""
    w = inputs.workload("cfg2", scen_ids=[3], n_req=1500)
    cap = 2000
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap)
    arr = w.traces.scenario(0)
    M = w.profile.M
    nd = int(o["stats"][0, 0])
    head = [0] * M
    states = []
    for k in range(nd):
        t = int(o["dec_t"][k])
        qs = []
        for m in range(M):
            tail = int(np.searchsorted(arr[m], t, side="right"))
            qs.append([t - int(a) for a in arr[m][head[m]:tail]])
        states.append(qs)
        head[int(o["dec_m"][k])] += int(o["dec_B"][k])
    q_off = [0]
    ws = []
    for qs in states:
        for q in qs:
            q_off.append(q_off[-1] + len(q))
            ws.extend(q)
    d = oracle.decide_batch(w.profile, w.cfgs, np.asarray(q_off, np.uint64), np.asarray(ws, np.uint32))
    assert np.array_equal(d["m"], o["dec_m"][:nd])
    assert np.array_equal(d["e"], o["dec_e"][:nd])
    assert np.array_equal(d["B"], o["dec_B"][:nd])
    assert np.array_equal(d["S"], o["dec_S"][:nd])


def _toy(seed, M, n):
    rng = np.random.default_rng(seed)
    return [sorted(rng.integers(0, 60000, size=rng.integers(0, n + 1)).tolist()) for _ in range(M)]


@pytest.mark.parametrize("seed", range(12))
def test_bruteforce_action_tree(seed):
    """Toy traces (M <= 3, <= 8 requests, E <= 3, B_max <= 3):
    (i) the independent mini-executor reproduces the greedy's completions from
    its action list; (ii) the tree minimum of violations is <= the greedy's;
    (iii) every greedy decision is the literal float64 Eq. 7 argmin among the
    Eq. 5-6 candidates (ties excepted)."""
    M = 2 + seed % 2
    prof = inputs.synth_profile(M, 3, [1, 2, 3], L_top=20000.0)
    tau = 30000
    arrivals = _toy(seed, M, 8 // M + 1)
    if sum(map(len, arrivals)) == 0:
        arrivals[0] = [0]
    tr = traces_from([arrivals])
    cfg = [inputs.SchedCfg(tau=tau, b_max=3, warmup=0)]
    o = oracle.replay_batch(prof, cfg, tr, dec_cap=64)
    nd = int(o["stats"][0, 0])
    actions = [(int(o["dec_m"][k]), int(o["dec_e"][k]), int(o["dec_B"][k])) for k in range(nd)]
    bs = list(prof.bs)
    comp = bf.mini_replay(arrivals, actions, lambda m, e, B: int(prof.lat[m, e, bs.index(B)]))
    flat = [c for q in comp for c in q]
    assert flat == o["completion"].tolist()
    best = bf.tree_min_violations(arrivals, prof, tau, 3)
    assert best <= int(o["stats"][0, 4])
    head = [0] * M
    for k in range(nd):
        t = int(o["dec_t"][k])
        qs = [[t - a for a in arrivals[m][head[m]:] if a <= t] for m in range(M)]
        ref = bf.literal_decide(prof, tau, 10, 3, qs)
        m_ref, e_ref, B_ref, scores = ref
        Ss = sorted(v[0] for v in scores.values())
        if not (len(Ss) > 1 and Ss[1] - Ss[0] < 1e-6 * max(1.0, Ss[0])):
            assert actions[k] == (m_ref, e_ref, B_ref)
        head[actions[k][0]] += actions[k][2]


def test_p95_golden():
    for ex in GOLD["p95"]:
        v = ex["values"]
        if v == "1..100":
            v = list(range(1, 101))
        elif v == "10,20,...,200":
            v = list(range(10, 201, 10))
        assert oracle.p95(v) == ex["p95"]


def test_violation_ratio_golden():
    """S:402-404 (Eq. 2, strict >) through replay on a 1-model line, L = 12 ms."""
    prof = prof1([12000])
    cfg = lambda tau: [inputs.SchedCfg(tau=tau, b_max=1, warmup=0)]
    iso = list(range(0, 20_000_000, 1_000_000))  # 20 isolated requests: T = 12000
    o = oracle.replay_batch(prof, cfg(12000), traces_from([[iso]]))
    assert np.all(o["lat"] == 12000) and int(o["stats"][0, 4]) == 0  # all T == tau -> V = 0
    o = oracle.replay_batch(prof, cfg(11999), traces_from([[iso]]))
    assert int(o["stats"][0, 4]) == 20  # all T > tau -> V = 1
    # 16 isolated + 4 simultaneous: T = 12, 24, 36, 48 ms in the burst -> 3 of 20
    arr = iso[:16] + [17_000_000] * 4
    o = oracle.replay_batch(prof, cfg(12000), traces_from([[arr]]))
    assert int(o["stats"][0, 4]) / int(o["stats"][0, 3]) == pytest.approx(0.15)


def test_group_stats_merge():
    w = inputs.workload("cfg2", scen_ids=np.arange(26), n_req=800)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces)
    cnt, p = oracle.group_stats(w.traces, o, w.cfgs, 13)
    for g in range(13):
        mem = np.nonzero(w.traces.group_id == g)[0]
        assert int(cnt[g, 4]) == int(o["stats"][mem, 4].sum())
        lats = np.concatenate([o["lat"][int(w.traces.arr_off[s * 4]) + 100:int(w.traces.arr_off[s * 4 + 4])]
                               for s in mem])
        assert int(p[g]) == int(np.sort(lats)[math.ceil(0.95 * lats.size) - 1])


def test_unsorted_arrivals_flagged():
    prof = prof1([1000])
    tr = traces_from([[[5, 3]]])
    o = oracle.replay_batch(prof, [inputs.SchedCfg(tau=50000, b_max=1)], tr)
    assert int(o["stats"][0, 7]) != 0
