"""Oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of EdgeServing's scheduler
(arxiv 2605.05527 §V, Algorithm 1) written straight from PAPER.md, used to
prove the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import it.  It shares no code with
paper_2605_05527_b200/ (no kernels, headers, tables, constants or helpers);
the only common module is ``inputs`` (seeded data generators, no arithmetic of
the method).

Functions and the passage each follows (P:n = PAPER.md line n):
  build_tables / H      reading Q5 of Eq. 3 in fixed point
  decide_batch          Algorithm 1 on queue snapshots: Eq. 5,
                        Eq. 6, prediction, Eq. 3-4,
                        Eq. 7
  replay_batch          online loop with exclusive time-division
                        execution; Eq. 1,
                        Eq. 2, warmup
  p95 / group_stats     nearest-rank P95 (reading Q15), per-group merge
  bruteforce.*          literal float64 Eq. 3-7 and full action-tree enumeration

Parity pins live in tests/test_oracle_*.py.  Unpinned parts: see DESIGN.md §5.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

F = 28  # fractional bits of the fixed-point score (reading Q5)
COLS = ["decisions", "candidates", "cells", "completed", "violations", "infeasible",
        "max_depth", "status", "sum_lat", "live", "terms", "acc_bp"] + [f"exit{e}" for e in range(8)]
NCOL = len(COLS)


def build(force=False):
    """Compile oracle.c with plain -O2 (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm", "-lpthread"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.or_H.restype = ctypes.c_uint64
            L.or_p95.restype = ctypes.c_uint32
            _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(0) if a is None else ctypes.c_void_p(a.ctypes.data)


def build_tables(tau: int, C: int = 10):
    """x_c, r, A, Bt and the min distance of any table value to an integer."""
    L = lib()
    cap = (tau * 4 >> 10) + 8
    A = np.zeros(cap, np.uint32)
    Bt = np.zeros(1024, np.uint32)
    xc = ctypes.c_uint64()
    r = ctypes.c_uint32()
    nA = ctypes.c_int()
    mg = ctypes.c_double()
    st = L.or_build_tables(ctypes.c_uint32(tau), ctypes.c_uint32(C), ctypes.byref(xc),
                           ctypes.byref(r), _p(A), ctypes.c_int(cap), ctypes.byref(nA), _p(Bt),
                           ctypes.byref(mg))
    if st:
        raise ValueError(f"or_build_tables status {st}")
    return {"x_c": int(xc.value), "r": int(r.value), "A": A[:nA.value].copy(), "Bt": Bt,
            "margin": float(mg.value), "C_q": C << F}


def H(tau: int, L_us: int):
    m = ctypes.c_double()
    v = lib().or_H(ctypes.c_uint32(tau), ctypes.c_uint32(L_us), ctypes.byref(m))
    return int(v), float(m.value)


def G(tables, w):
    """G(w) = (A[(w+r)>>10] * Bt[(w+r)&1023]) >> F for 0 <= w < x_c (reading Q5)."""
    w = np.asarray(w, dtype=np.uint64)
    v = w + np.uint64(tables["r"])
    a = tables["A"][(v >> np.uint64(10)).astype(np.int64)].astype(np.uint64)
    b = tables["Bt"][(v & np.uint64(1023)).astype(np.int64)].astype(np.uint64)
    return (a * b) >> np.uint64(F)


def validate_profile(prof):
    bad = np.zeros(3, np.int32)
    st = lib().or_validate_profile(prof.M, prof.E, prof.nb, _p(np.ascontiguousarray(prof.bs, np.int32)),
                                   _p(np.ascontiguousarray(prof.lat, np.uint32)),
                                   _p(np.ascontiguousarray(prof.mask, np.uint8)), _p(bad))
    return int(st), tuple(int(x) for x in bad)


# selection policies (oracle.c OR_POL_*, Q26)
POLICIES = {"edgeserving": 0, "all_final": 1, "all_early": 2, "ee_lqf": 3, "ee_edf": 4, "allfinal_da": 5,
            "ours_bs1": 6, "symphony": 7, "grid": 8}


def _cfg_arrays(cfgs):
    tau = np.array([c.tau for c in cfgs], np.uint32)
    C = np.array([c.C for c in cfgs], np.uint32)
    bm = np.array([c.b_max for c in cfgs], np.uint32)
    wu = np.array([c.warmup for c in cfgs], np.uint32)
    pol = np.array([getattr(c, "policy", 0) for c in cfgs], np.uint32)
    return tau, C, bm, wu, pol


def decide_batch(prof, cfgs, q_off, waits, cfg_idx=None):
    """Algorithm 1 on n snapshots (CSR q_off[n*M+1] into head-first waits)."""
    M = prof.M
    q_off = np.ascontiguousarray(q_off, np.uint64)
    waits = np.ascontiguousarray(waits, np.uint32)
    n = (q_off.size - 1) // M
    tau, C, bm, _, pol = _cfg_arrays(cfgs)
    ci = None if cfg_idx is None else np.ascontiguousarray(cfg_idx, np.uint16)
    out = {"m": np.zeros(n, np.uint8), "e": np.zeros(n, np.uint8), "B": np.zeros(n, np.uint16),
           "L": np.zeros(n, np.uint32), "S": np.zeros(n, np.uint64), "flags": np.zeros(n, np.uint8),
           "cand": np.zeros(n * M, np.uint64), "cand_dbl": np.zeros(n * M, np.float64)}
    bs = np.ascontiguousarray(prof.bs, np.int32)
    lat = np.ascontiguousarray(prof.lat, np.uint32)
    mask = np.ascontiguousarray(prof.mask, np.uint8)
    st = lib().or_decide_batch(
        M, prof.E, prof.nb, _p(bs), _p(lat), _p(mask), _p(tau), _p(C), _p(bm), _p(pol), len(cfgs),
        ctypes.c_int64(n), _p(ci), _p(q_off), _p(waits), _p(out["m"]), _p(out["e"]), _p(out["B"]),
        _p(out["L"]), _p(out["S"]), _p(out["flags"]), _p(out["cand"]), _p(out["cand_dbl"]))
    if st:
        raise ValueError(f"or_decide_batch status {st}")
    out["cand"] = out["cand"].reshape(n, M)
    out["cand_dbl"] = out["cand_dbl"].reshape(n, M)
    return out


def replay_batch(prof, cfgs, traces, full=True, dec_cap=0, nthreads=1):
    """Replay every scenario of ``traces`` (inputs.Traces) decision by decision."""
    M = prof.M
    n = traces.n_scen
    total = int(traces.arr_off[-1])
    tau, C, bm, wu, pol = _cfg_arrays(cfgs)
    arr_off = np.ascontiguousarray(traces.arr_off, np.uint64)
    arrival = np.ascontiguousarray(traces.arrival, np.uint32)
    ci = np.ascontiguousarray(traces.cfg_idx, np.uint16)
    out = {"stats": np.zeros((n, NCOL), np.uint64), "p95": np.zeros(n, np.uint32)}
    if full:
        out["completion"] = np.zeros(total, np.uint32)
        out["exit"] = np.zeros(total, np.uint8)
        out["lat"] = np.zeros(total, np.uint32)
    if dec_cap:
        out["dec_t"] = np.zeros(n * dec_cap, np.uint32)
        out["dec_m"] = np.zeros(n * dec_cap, np.uint8)
        out["dec_e"] = np.zeros(n * dec_cap, np.uint8)
        out["dec_B"] = np.zeros(n * dec_cap, np.uint16)
        out["dec_L"] = np.zeros(n * dec_cap, np.uint32)
        out["dec_S"] = np.zeros(n * dec_cap, np.uint64)
        out["dec_f"] = np.zeros(n * dec_cap, np.uint8)
    bs = np.ascontiguousarray(prof.bs, np.int32)
    lat = np.ascontiguousarray(prof.lat, np.uint32)
    mask = np.ascontiguousarray(prof.mask, np.uint8)
    acc = getattr(prof, "acc", None)
    acc = None if acc is None else np.ascontiguousarray(acc, np.uint16)
    g = out.get
    st = lib().or_replay_batch(
        M, prof.E, prof.nb, _p(bs), _p(lat), _p(mask), _p(acc), _p(tau), _p(C), _p(bm), _p(wu), _p(pol), len(cfgs),
        ctypes.c_int64(n), _p(ci), _p(arr_off), _p(arrival), _p(g("completion")), _p(g("exit")),
        _p(g("lat")), _p(out["stats"]), _p(out["p95"]), ctypes.c_int64(dec_cap), _p(g("dec_t")),
        _p(g("dec_m")), _p(g("dec_e")), _p(g("dec_B")), _p(g("dec_L")), _p(g("dec_S")),
        _p(g("dec_f")), ctypes.c_int(nthreads))
    if st:
        raise ValueError(f"or_replay_batch status {st}")
    return out


GROUP_COLS = ["decisions", "candidates", "cells", "completed", "violations", "infeasible", "sum_lat",
              "acc_bp"] + [f"exit{e}" for e in range(8)]
GROUP_SRC = [COLS.index(c) for c in GROUP_COLS]


def p95(values):
    """Nearest-rank P95: the ceil(0.95 N)-th smallest (reading Q15)."""
    v = np.ascontiguousarray(values, np.uint32)
    return int(lib().or_p95(_p(v), ctypes.c_int64(v.size)))


def group_stats(traces, out, cfgs, n_groups):
    """Per-group merge (north star): summed counters and the exact nearest-rank
    P95 over the union of every member scenario's post-warmup latencies."""
    G_ = n_groups
    stats = out["stats"]
    cnt = np.zeros((G_, len(GROUP_COLS)), np.uint64)
    p = np.zeros(G_, np.uint32)
    lats = [[] for _ in range(G_)]
    M = traces.M
    for s in range(traces.n_scen):
        g = int(traces.group_id[s])
        cnt[g] += stats[s][GROUP_SRC]
        lo = int(traces.arr_off[s * M])
        hi = int(traces.arr_off[s * M + M])
        W = cfgs[int(traces.cfg_idx[s])].warmup
        if hi - lo > W:
            lats[g].append(out["lat"][lo + W:hi])
    for g in range(G_):
        if lats[g]:
            p[g] = p95(np.concatenate(lats[g]))
    return cnt, p
