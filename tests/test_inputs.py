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
