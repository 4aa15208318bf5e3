"""Pins of the oracle's fixed-point urgency tables (reading Q5 of Eq. 3).

Each test checks the oracle against something other than itself: the paper's
closed forms (f(tau) = exp(0) = 1; clip at tau(1 + ln C)), the
SPEC worked examples (tests/golden/spec_examples.json) and Python's float64
math.exp as an independent evaluation of exp.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
F = 28
TAUS = [1024, 20000, 50000, 100000, 1 << 20]
CS = [1, 2, 10, 15]


@pytest.mark.parametrize("tau", TAUS)
@pytest.mark.parametrize("C", CS)
def test_clip_boundary_closed_form(tau, C):
    """x_c = ceil(tau(1 + ln C)) (reading Q6); C = 1 gives tau exactly."""
    t = oracle.build_tables(tau, C)
    y = tau * (1.0 + math.log(C))
    assert t["x_c"] == math.ceil(y)
    if C == 1:
        assert t["x_c"] == tau
    # the integer boundary really separates clipped from unclipped
    assert math.exp((t["x_c"] - 1) / tau - 1.0) < C <= math.exp(t["x_c"] / tau - 1.0) + 1e-12


def test_clip_boundary_golden():
    g = GOLD["clip_boundary"]
    assert oracle.build_tables(g["tau_us"], g["C"])["x_c"] == g["x_c"]


@pytest.mark.parametrize("tau", TAUS)
@pytest.mark.parametrize("C", CS)
def test_G_at_tau_is_exactly_one(tau, C):
    """f(tau) = exp(0) = 1 for every SLO: G(tau) = 2^F exactly."""
    t = oracle.build_tables(tau, C)
    if tau < t["x_c"]:
        assert int(oracle.G(t, [tau])[0]) == 1 << F
    assert oracle.H(tau, 0)[0] == 1 << F  # exp(0 / tau) = 1


@pytest.mark.parametrize("tau", [20000, 50000, 100000])
def test_G_matches_float_exp_everywhere(tau):
    """|G(w) 2^-F - exp((w - tau)/tau)| stays within the floor-error bound for
    every 0 <= w < x_c: with a >= A - 1, b >= Bt - 1, a*b >= A*Bt - A - Bt, so
    the error is < (A + Bt)/2^F + 1 <= C + exp(1023/tau) + 1 quanta."""
    t = oracle.build_tables(tau, 10)
    w = np.arange(t["x_c"], dtype=np.uint64)
    g = oracle.G(t, w).astype(np.float64)
    ref = np.exp((w.astype(np.float64) - tau) / tau) * 2.0 ** F
    err = np.abs(g - ref)
    assert err.max() <= 10 + math.exp(1023 / tau) + 1
    assert np.all(g <= ref + 1e-3)  # every floor is <= the true value
    assert np.all(np.diff(g) > 0)  # strictly increasing (>= 987 quanta/us at tau=100ms)


@pytest.mark.parametrize("tau", TAUS)
@pytest.mark.parametrize("C", CS)
def test_tables_fit_and_floor_is_unambiguous(tau, C):
    """A, Bt, G < 2^32; the real table values stay >= 1e-7 from an integer, so
    their floor is fixed far beyond long-double expl error (~1e-9 absolute)."""
    t = oracle.build_tables(tau, C)
    assert t["A"].max() < 2 ** 32 and t["Bt"].max() < 2 ** 32
    assert int(t["A"][-1]) < C << F  # A < C 2^F by construction of x_c
    assert t["margin"] > 1e-7
    # A and Bt against float64 exp, element by element
    h = np.arange(t["A"].size)
    refA = np.exp((h * 1024.0 - t["r"] - tau) / tau) * 2.0 ** F
    assert np.all(np.abs(t["A"] - np.floor(refA)) <= 1)
    refB = np.exp(np.arange(1024) / tau) * 2.0 ** F
    assert np.all(np.abs(t["Bt"] - np.floor(refB)) <= 1)
    assert (tau + t["r"]) % 1024 == 0


def test_urgency_golden():
    """S:189-192 urgency values through G (unclipped) and the clip."""
    tau = 50000
    t = oracle.build_tables(tau, 10)
    for ex in GOLD["urgency"]:
        w = int(round(ex["w_over_tau"] * tau))
        if w >= t["x_c"]:
            val = 10.0  # clipped: contributes C
        else:
            val = int(oracle.G(t, [w])[0]) / 2.0 ** F
        assert abs(val - ex["f"]) < 1e-6


def test_H_values():
    """H(L) = floor(2^F exp(L/tau)) needs 33 bits below x_c (u64 in both sides)."""
    tau = 50000
    t = oracle.build_tables(tau, 10)
    for L in [1, 1000, 12000, 30000, t["x_c"] - 1]:
        h, mg = oracle.H(tau, L)
        assert abs(h - math.exp(L / tau) * 2 ** F) <= 1.0
        assert mg > 1e-7
    assert oracle.H(tau, t["x_c"] - 1)[0] >= 2 ** 32


def test_out_of_range_rejected():
    for tau, C in [(1023, 10), ((1 << 20) + 1, 10), (50000, 0), (50000, 16)]:
        with pytest.raises(ValueError):
            oracle.build_tables(tau, C)
