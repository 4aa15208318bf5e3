"""The seeded input generators (inputs/): determinism, subset independence,
the Fig. profile_mean laws of the synthetic profile and
arrival-process moments (MMPP mean-rate preservation)."""
import math

import numpy as np
import pytest

import inputs
import oracle


def test_profile_laws_and_validity():
    for (M, E, bs) in [(3, 3, [1, 2, 4, 8]), (4, 4, list(range(1, 17))), (8, 5, list(range(1, 33)))]:
        p = inputs.synth_profile(M, E, bs)
        assert oracle.validate_profile(p)[0] == 0
        lat = p.lat.astype(np.float64)
        r_b = lat[:, :, -1] / lat[:, :, 0]
        assert np.all((r_b >= 2.0) & (r_b <= 3.0))  # batch 1 -> B_max: 2-3x
        r_e = lat[:, -1, :] / lat[:, 0, :]
        assert np.all((r_e >= 6.0) & (r_e <= 8.0))  # final ~6-8x layer1
        assert np.all(np.diff(lat, axis=0) > 0)  # heavier models slower
        assert p.lat[M - 1, E - 1, 0] == 12000


def test_profile_validation_names_cell():
    p = inputs.synth_profile(3, 3, [1, 2, 4, 8])
    bad = p.lat.copy()
    bad[1, 2, 0] = bad[1, 1, 0]  # not strictly increasing in exit
    st, cell = oracle.validate_profile(inputs.Profile(3, 3, p.bs, bad, p.mask))
    assert st == 2 and cell == (1, 2, 0)


def test_determinism_and_subset_independence():
    a = inputs.workload("cfg2", scen_ids=[0, 1, 2, 3], n_req=500)
    b = inputs.workload("cfg2", scen_ids=[2, 3], n_req=500)
    for k in range(2):
        for m in range(4):
            assert np.array_equal(a.traces.scenario(2 + k)[m], b.traces.scenario(k)[m])
    c = inputs.workload("cfg2", scen_ids=[0, 1, 2, 3], n_req=500)
    assert np.array_equal(a.traces.arrival, c.traces.arrival)


def test_poisson_moments():
    lam = 0.002  # per us
    segs = inputs.poisson_segments(3, np.arange(64), np.full((64, 1), lam), np.full(64, 1e6))
    counts = np.array([s[0].size for s in segs])
    assert abs(counts.mean() - 2000) < 4 * math.sqrt(2000 / 64)
    gaps = np.concatenate([np.diff(s[0].astype(np.float64)) for s in segs])
    assert abs(gaps.mean() - 500.0) < 10.0
    assert abs(gaps.std() / gaps.mean() - 1.0) < 0.05  # exponential: CV = 1


def test_mmpp_preserves_mean_rate_and_is_bursty():
    lam = np.full((32, 1), 0.001)
    D = np.full(32, 2e7)
    segs = inputs.mmpp_segments(9, np.arange(32), lam, D)
    counts = np.array([s[0].size for s in segs])
    assert abs(counts.mean() / 20000 - 1.0) < 0.1
    # index of dispersion of counts in 50 ms windows >> 1 (Poisson would give 1)
    a = segs[0][0]
    h = np.bincount((a // 50000).astype(np.int64))
    assert h.var() / h.mean() > 3.0


def test_snapshot_generators_are_fifo():
    q_off, w = inputs.snapshots_poisson_depth(1, np.arange(16), 4, 300, [0.001] * 4)
    for s in range(16 * 4):
        q = w[q_off[s]:q_off[s + 1]]
        assert np.all(np.diff(q.astype(np.int64)) <= 0)


def test_harvest_snapshots_matches_plain_loop():
    """The vectorised harvest equals a plain per-decision loop (searchsorted
    tail, head advanced by the dispatched batch) on a hand-made decision log."""
    M = 3
    per = [[np.array([0, 5, 9, 12, 30], np.uint32), np.array([2, 3], np.uint32), np.array([], np.uint32)],
           [np.array([1], np.uint32), np.array([4, 4, 8, 20], np.uint32), np.array([0, 7], np.uint32)]]
    tr = inputs._assemble(M, per, np.array([0, 1], np.uint16), np.array([0, 0], np.uint32), np.arange(2))
    cap = 4
    n_dec = np.array([3, 4])
    dec_t = np.array([3, 10, 31, 0, 1, 8, 9, 25], np.uint32)
    dec_m = np.array([1, 0, 0, 0, 2, 1, 0, 1], np.uint8)
    dec_B = np.array([2, 2, 3, 0, 1, 2, 1, 2], np.uint16)
    q, w, ci = inputs.harvest_snapshots(tr, n_dec, cap, dec_t, dec_m, dec_B)
    ref_q, ref_w = [0], []
    for s in range(2):
        arr = tr.scenario(s)
        head = [0] * M
        for k in range(int(n_dec[s])):
            t = int(dec_t[s * cap + k])
            for m in range(M):
                tail = int(np.searchsorted(arr[m], t, side="right"))
                ref_w.extend(t - int(a) for a in arr[m][head[m]:tail])
                ref_q.append(len(ref_w))
            head[int(dec_m[s * cap + k])] += int(dec_B[s * cap + k])
    assert q.tolist() == ref_q and w.tolist() == ref_w
    assert ci.tolist() == [0, 0, 0, 1, 1, 1, 1]
    # snapshot 0 of scenario 0 at t=3: Q0 = {0}, Q1 = {2, 3}, Q2 = {} -> waits 3 | 1 0
    assert w[:3].tolist() == [3, 1, 0] and q[1:4].tolist() == [1, 3, 3]
