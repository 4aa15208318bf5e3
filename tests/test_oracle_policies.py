"""Pins of the oracle's baseline / ablation policies (Q26): the
paper's All-Final / All-Early (§VI-A) and Early-Exit+LQF,
Early-Exit+EDF, All-Final+Deadline-Aware, Ours+bs=1 (§VI-H).

Pinned by the SPEC worked examples of policy_decide, by an
independent float64 brute force written from the paper's one-line
definitions (oracle/bruteforce.literal_policy_decide) on seeded random
states, and by the invariants S:295-298 (LQF ties -> lowest model; exits of
ee_lqf / ee_edf equal Eq. 6 for the chosen queue; all_final / allfinal_da
always report the deepest exit).
"""
import numpy as np
import pytest

import inputs
import oracle
from oracle import bruteforce as bf

F = 28
POL = oracle.POLICIES


def snap(queues):
    q_off = np.zeros(len(queues) + 1, np.uint64)
    q_off[1:] = np.cumsum([len(q) for q in queues])
    w = np.concatenate([np.asarray(q, np.uint32) for q in queues]) if sum(map(len, queues)) else \
        np.zeros(0, np.uint32)
    return q_off, w


def one(prof, policy, queues, tau=50000, b_max=8):
    q_off, w = snap(queues)
    return oracle.decide_batch(prof, [inputs.SchedCfg(tau=tau, b_max=b_max, policy=POL[policy])], q_off, w)


def test_spec_examples():
    prof = inputs.synth_profile(3, 3, [1, 2, 4, 8])
    # ee_lqf with queue lengths {3, 7, 5} -> the model with length 7
    o = one(prof, "ee_lqf", [[100] * 3, [100] * 7, [100] * 5])
    assert int(o["m"][0]) == 1
    # ee_edf with oldest waits {10, 40, 25} ms, tau = 50 ms -> the 40 ms queue (slack 10 ms)
    o = one(prof, "ee_edf", [[10000], [40000], [25000]])
    assert int(o["m"][0]) == 1


def test_ties_and_fixed_exits():
    prof = inputs.synth_profile(3, 4, [1, 2, 4, 8])
    for pol in ["all_final", "all_early", "ee_lqf"]:
        o = one(prof, pol, [[], [900, 800], [5, 4]])  # equal lengths: lowest model
        assert int(o["m"][0]) == 1
    o = one(prof, "ee_edf", [[7000, 1], [7000], []])  # equal head waits: lowest model
    assert int(o["m"][0]) == 0
    mask = np.ones((3, 4), np.uint8)
    mask[1, 3] = 0  # model 1: final exit disallowed -> deepest allowed is 2
    mask[1, 0] = 0  # shallowest allowed is 1
    pm = inputs.Profile(M=3, E=4, bs=prof.bs, lat=prof.lat, mask=mask)
    for pol, e in [("all_final", 2), ("allfinal_da", 2), ("all_early", 1)]:
        o = one(pm, pol, [[], [10, 9, 8], []])
        assert int(o["m"][0]) == 1 and int(o["e"][0]) == e
        L = int(prof.lat[1, e, 2])  # B = 3 -> profiled 2 (index 1)? use the oracle's B
        bi = list(prof.bs).index(int(o["B"][0]))
        assert int(o["L"][0]) == int(prof.lat[1, e, bi])
        assert bool(o["flags"][0] & 1) == (10 + int(prof.lat[1, e, bi]) <= 50000)
    o = one(prof, "ours_bs1", [[40000] * 6, [30000] * 8, [1]])
    assert int(o["B"][0]) == 1
    # LQF / EDF policies score nothing
    o = one(prof, "ee_lqf", [[1, 0], [3], []])
    assert int(o["S"][0]) == 0 and np.all(o["cand"] == np.iinfo(np.uint64).max)


def _states(n, M, max_len, tau, seed):
    q_off, w = inputs.snapshots_uniform(seed, n, M, max_len, 3 * tau)
    st = [[list(map(int, w[q_off[s * M + m]:q_off[s * M + m + 1]])) for m in range(M)] for s in range(n)]
    return q_off, w, st


@pytest.mark.parametrize("policy", [p for p in POL if p not in ("symphony", "grid")])
def test_policies_vs_literal_bruteforce(policy):
    """600 seeded random states per policy (queues <= 10, waits in [0, 3 tau],
    sparse batch grid, one model with a restricted exit mask): model, exit,
    batch and feasibility equal the literal float64 reading; scoring policies
    agree with the float64 score within the Q5 error bound, argmin exact
    except on float near-ties."""
    tau, M = 50000, 3
    base = inputs.synth_profile(M, 4, [1, 2, 4, 8], L_top=20000.0)
    mask = np.ones((M, 4), np.uint8)
    mask[2, 3] = 0
    mask[2, 0] = 0
    prof = inputs.Profile(M=M, E=4, bs=base.bs, lat=base.lat, mask=mask)
    cfg = [inputs.SchedCfg(tau=tau, b_max=6, policy=POL[policy])]
    q_off, w, states = _states(600, M, 10, tau, seed=500 + POL[policy])
    o = oracle.decide_batch(prof, cfg, q_off, w)
    near = 0
    for s, qs in enumerate(states):
        ref = bf.literal_policy_decide(prof, tau, 10, 6, qs, policy)
        if ref is None:
            assert o["flags"][s] == 2
            continue
        m_ref, e_ref, B_ref, feas_ref, scores = ref
        for m, S in scores.items():
            assert abs(int(o["cand"][s, m]) / 2.0 ** F - S) <= 1e-6 * max(1.0, S) + 1e-6
        if len(scores) > 1:
            Ss = sorted(scores.values())
            if Ss[1] - Ss[0] < 1e-5 * max(1.0, Ss[0]):
                near += 1
                continue
        assert int(o["m"][s]) == m_ref, (s, qs)
        assert (int(o["e"][s]), int(o["B"][s]), bool(o["flags"][s] & 1)) == (e_ref, B_ref, feas_ref), (s, qs)
    assert near < 20


def test_policy_exits_equal_eq6_of_chosen_queue():
    """ee_lqf / ee_edf exits equal the EdgeServing Eq. 6 choice for the
    queue they pick (checked against the pinned EdgeServing oracle on the
    chosen queue alone: Eq. 5/6 depend on that queue only)."""
    tau, M = 50000, 4
    prof = inputs.synth_profile(M, 4, list(range(1, 11)))
    q_off, w, states = _states(300, M, 10, tau, seed=91)
    for pol in ["ee_lqf", "ee_edf"]:
        o = oracle.decide_batch(prof, [inputs.SchedCfg(tau=tau, b_max=10, policy=POL[pol])], q_off, w)
        for s, qs in enumerate(states):
            if o["flags"][s] & 2:
                continue
            m = int(o["m"][s])
            alone = [q if i == m else [] for i, q in enumerate(qs)]
            r = one(prof, "edgeserving", alone, tau=tau, b_max=10)
            assert (int(r["e"][0]), int(r["B"][0]), int(r["flags"][0])) == \
                (int(o["e"][s]), int(o["B"][s]), int(o["flags"][s]))


@pytest.mark.parametrize("policy", list(POL))
def test_policy_replay_invariants(policy):
    """Replays under every policy keep the executor invariants (conservation,
    every request served once, S:298 exits, bs=1 batches)."""
    w = inputs.workload("cfg1", n_req=600)
    cfgs = [inputs.SchedCfg(tau=c.tau, b_max=c.b_max, policy=POL[policy]) for c in w.cfgs]
    o = oracle.replay_batch(w.profile, cfgs, w.traces, dec_cap=2000)
    st = o["stats"][0]
    n = int(w.traces.arr_off[-1])
    assert int(st[7]) == 0 and int(st[3]) == n - 100
    assert np.all(o["completion"] >= w.traces.arrival)
    d = int(st[0])
    if policy in ("all_final", "allfinal_da"):
        assert np.all(o["dec_e"][:d] == w.profile.E - 1) and np.all(o["exit"] == w.profile.E - 1)
    if policy == "all_early":
        assert np.all(o["dec_e"][:d] == 0)
    if policy == "ours_bs1":
        assert np.all(o["dec_B"][:d] == 1) and d == n
    if POL[policy] in (1, 2, 3, 4):
        assert np.all(o["dec_S"][:d] == 0) and int(st[10]) == 0  # no Eq. 4 terms


def _toy_traces(seed, M, n, span):
    rng = np.random.default_rng(seed)
    arr = [sorted(int(x) for x in rng.integers(0, span, rng.integers(1, n + 1))) for _ in range(M)]
    off = np.zeros(M + 1, np.uint64)
    off[1:] = np.cumsum([len(a) for a in arr])
    tr = inputs.Traces(M=M, arr_off=off, arrival=np.concatenate([np.asarray(a, np.uint32) for a in arr]),
                       cfg_idx=np.zeros(1, np.uint16), group_id=np.zeros(1, np.uint32))
    return arr, tr


def test_symphony_spec_example():
    """single queue, oldest wait 10 ms, L(final, B) = 28 ms, tau = 50 ms
    -> the dispatch waits 12 ms more: the request starts at a + 22 ms and
    completes at a + 50 ms (T = tau, not a violation, Q16)."""
    lat = np.array([[[9000, 12000], [28000, 40000]]], np.uint32)  # 1 model, exits {layer1, final}, batch {1, 2}
    prof = inputs.Profile(M=1, E=2, bs=np.array([1, 2], np.int32), lat=lat, mask=np.ones((1, 2), np.uint8))
    arr, tr = [[1000]], inputs.Traces(M=1, arr_off=np.array([0, 1], np.uint64), arrival=np.array([1000], np.uint32),
                                      cfg_idx=np.zeros(1, np.uint16), group_id=np.zeros(1, np.uint32))
    cfg = [inputs.SchedCfg(tau=50000, b_max=2, warmup=0, policy=POL["symphony"])]  # one task < B_max: defer
    o = oracle.replay_batch(prof, cfg, tr, dec_cap=4)
    assert int(o["dec_t"][0]) == 1000 + 22000 and int(o["dec_e"][0]) == 1
    assert int(o["completion"][0]) == 1000 + 50000 and int(o["stats"][0][4]) == 0


@pytest.mark.parametrize("seed", range(12))
def test_symphony_vs_microsecond_simulation(seed):
    """The oracle's event-jump Symphony replay (wake at the earliest trigger or
    arrival) equals a microsecond-by-microsecond simulation of the same rule
    (bruteforce.symphony_replay_us) on toy traces: every dispatch (t, m, e,
    B) and every completion time."""
    M = 1 + seed % 3
    prof = inputs.synth_profile(M, 3, [1, 2, 4], L_top=9000.0)
    arr, tr = _toy_traces(seed, M, 7, 60000)
    tau, b_max = 20000 + 2000 * seed, 4
    cfg = [inputs.SchedCfg(tau=tau, b_max=b_max, warmup=0, policy=POL["symphony"])]
    o = oracle.replay_batch(prof, cfg, tr, dec_cap=64)
    ref, done = bf.symphony_replay_us(prof, tau, b_max, arr)
    d = int(o["stats"][0][0])
    assert d == len(ref)
    got = [(int(o["dec_t"][k]), int(o["dec_m"][k]), int(o["dec_e"][k]), int(o["dec_B"][k])) for k in range(d)]
    assert got == ref
    assert o["completion"].tolist() == [x for q in done for x in q]


def test_symphony_never_dispatches_early():
    """a dispatched batch's head would miss tau after one more idle
    microsecond (w_head + L >= tau), unless its queue had reached B_max."""
    w = inputs.workload("cfg2", scen_ids=[0, 5, 12], n_req=1500)
    cfgs = [inputs.SchedCfg(tau=c.tau, b_max=c.b_max, policy=POL["symphony"]) for c in w.cfgs]
    o = oracle.replay_batch(w.profile, cfgs, w.traces, dec_cap=2000)
    M = w.profile.M
    for s in range(3):
        arr = [w.traces.arrival[int(w.traces.arr_off[s * M + m]):int(w.traces.arr_off[s * M + m + 1])]
               for m in range(M)]
        head = [0] * M
        for k in range(int(o["stats"][s][0])):
            t, m, B, L = (int(o[x][s * 2000 + k]) for x in ("dec_t", "dec_m", "dec_B", "dec_L"))
            q = int(np.searchsorted(arr[m], t, side="right")) - head[m]
            assert t - int(arr[m][head[m]]) + L >= cfgs[0].tau or q >= cfgs[0].b_max
            assert int(o["dec_e"][s * 2000 + k]) == w.profile.E - 1
            head[m] += B


def test_grid_vs_literal_bruteforce():
    """GRID (f2): 400 seeded states, every admissible (m, e, b) scored; the
    oracle's (m, e, b, feasible) equals the literal float64 argmin of
    (S, m, e, b) except on float near-ties; per-model best scores within the
    Q5 bound; GRID never picks a deeper exit than the shallowest allowed one
    for its (m, b) (S is non-decreasing in L, L strictly increasing in e)."""
    tau, M = 50000, 3
    base = inputs.synth_profile(M, 4, [1, 2, 4, 8], L_top=20000.0)
    mask = np.ones((M, 4), np.uint8)
    mask[1, 0] = 0
    prof = inputs.Profile(M=M, E=4, bs=base.bs, lat=base.lat, mask=mask)
    cfg = [inputs.SchedCfg(tau=tau, b_max=6, policy=POL["grid"])]
    q_off, w, states = _states(400, M, 10, tau, seed=808)
    o = oracle.decide_batch(prof, cfg, q_off, w)
    near = 0
    for s, qs in enumerate(states):
        ref = bf.literal_grid_decide(prof, tau, 10, 6, qs)
        if ref is None:
            assert o["flags"][s] == 2
            continue
        m_ref, e_ref, b_ref, feas_ref, scores = ref
        for m in range(M):
            sm = [v for k, v in scores.items() if k[0] == m]
            if sm:
                assert abs(int(o["cand"][s, m]) / 2.0 ** F - min(sm)) <= 1e-6 * max(1.0, min(sm)) + 1e-6
        Ss = sorted(scores.values())
        if len(Ss) > 1 and Ss[1] - Ss[0] < 1e-5 * max(1.0, Ss[0]):
            near += 1
            continue
        assert (int(o["m"][s]), int(o["e"][s]), int(o["B"][s]), bool(o["flags"][s] & 1)) == \
            (m_ref, e_ref, b_ref, feas_ref), (s, qs)
        assert int(o["e"][s]) == min(e for e in range(4) if mask[m_ref][e])
    assert near < 40
