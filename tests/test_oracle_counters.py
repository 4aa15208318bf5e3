"""Pins of the oracle's replay work counters (decisions, candidates, cells,
live, terms, max depth, infeasible) and of a GRID decision's admissible-cell
count, against replays computed by hand in tests/golden/work_counters.json
(each case carries its derivation).  The same golden cases run through the
GPU replay in tests/test_gpu_parity.py::test_k2_golden_work_counters."""
import json
import os

import numpy as np
import pytest

import inputs
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "work_counters.json")))
COLS = ["decisions", "candidates", "cells", "completed", "violations", "infeasible", "max_depth", "status",
        "sum_lat", "live", "terms", "acc_bp"]


def golden_case(case):
    p = case["profile"]
    p = GOLD[p] if isinstance(p, str) else p
    lat = np.asarray(p["lat"], np.uint32)
    prof = inputs.Profile(M=p["M"], E=p["E"], bs=np.asarray(p["bs"], np.int32), lat=lat,
                          mask=np.ones((p["M"], p["E"]), np.uint8),
                          acc=np.asarray(p["acc"], np.uint16) if "acc" in p else None)
    c = case["cfg"]
    cfgs = [inputs.SchedCfg(tau=c["tau"], b_max=c["b_max"], C=c["C"], warmup=c["warmup"], policy=c["policy"])]
    segs = [[np.asarray(a, np.uint32) for a in case["arrivals"]]]
    tr = inputs._assemble(p["M"], segs, [0], [0], np.arange(1))
    return prof, cfgs, tr


def expected_row(case):
    st = case["stats"]
    ex = list(st["exit"]) + [0] * (8 - len(st["exit"]))
    return np.array([st.get(k, 0) for k in COLS] + ex, np.uint64)


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"][:40] for c in GOLD["cases"]])
def test_oracle_work_counters_hand_computed(case):
    prof, cfgs, tr = golden_case(case)
    o = oracle.replay_batch(prof, cfgs, tr, full=True)
    assert np.array_equal(o["stats"][0], expected_row(case)), (o["stats"][0], expected_row(case))
    assert np.array_equal(o["lat"], np.asarray(case["latency"], np.uint32))
    assert int(o["p95"][0]) == case["p95"]
