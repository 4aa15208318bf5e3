"""Thin Python binding of libedgeserve.so (include/edgeserve.h).

Argument marshalling only: every step of the stability-score path runs in the
CUDA kernels behind the C ABI.  Device buffers are torch tensors (PyTorch is
used for device memory and streams only); there is no CPU fallback -- calls
raise if the shared library or a CUDA device is missing.

Functions keep the C names: es_load_profile, es_score_candidates,
es_replay_traces, es_replay_traces_host, es_group_accumulate, es_group_hist,
es_group_p95_select, es_device_status, es_get_tables.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ES_LIB") or os.path.join(_HERE, "libedgeserve.so")

ES_NSTAT = 20
ES_NGSTAT = 16
ES_HIST_BINS = 4096
STAT_COLS = ["decisions", "candidates", "cells", "completed", "violations", "infeasible", "max_depth",
             "status", "sum_lat", "live", "terms", "acc_bp"] + [f"exit{e}" for e in range(8)]
GROUP_COLS = ["decisions", "candidates", "cells", "completed", "violations", "infeasible", "sum_lat",
              "acc_bp"] + [f"exit{e}" for e in range(8)]
STATUS = {0: "ES_OK", 1: "ES_ERR_ARG", 2: "ES_ERR_PROFILE_GRID", 3: "ES_ERR_PROFILE_MONOTONE",
          4: "ES_ERR_OUT_OF_GRID", 5: "ES_ERR_RANGE", 6: "ES_ERR_CUDA", 7: "ES_ERR_OOM",
          8: "ES_ERR_UNSORTED", 9: "ES_ERR_NUMERIC", 10: "ES_ERR_INTERNAL"}
EXPORTS = ["es_last_error", "es_version", "es_load_profile", "es_free_profile", "es_get_tables",
           "es_score_candidates", "es_replay_traces", "es_scen_p95", "es_scen_stats", "es_replay_traces_host",
           "es_replay_traces_host_pipelined",
           "es_group_accumulate",
           "es_group_hist", "es_group_p95_select", "es_device_status", "es_launch_count"]

P = ctypes.c_void_p


class ProfileDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("E", ctypes.c_int32), ("nb", ctypes.c_int32),
                ("batch_sizes", P), ("latency_us", P), ("exit_mask", P), ("accuracy_bp", P)]


class SchedCfg(ctypes.Structure):
    _fields_ = [("tau_us", ctypes.c_uint32), ("clip_C", ctypes.c_uint32), ("b_max", ctypes.c_uint32),
                ("warmup", ctypes.c_uint32), ("policy", ctypes.c_uint32)]


class Snapshots(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("cfg_idx", P), ("q_off", P), ("waits_us", P), ("n_waits", ctypes.c_int64)]


class Decisions(ctypes.Structure):
    _fields_ = [("m", P), ("e", P), ("B", P), ("L_us", P), ("score_q", P), ("flags", P),
                ("cand_score_q", P)]


class Traces(ctypes.Structure):
    _fields_ = [("n_scen", ctypes.c_int64), ("cfg_idx", P), ("group_id", P), ("arr_off", P),
                ("arrival_us", P)]


class ReplayOut(ctypes.Structure):
    _fields_ = [("completion_us", P), ("exit_used", P), ("latency_us", P), ("scen_stats", P),
                ("scen_p95_us", P), ("dec_cap", ctypes.c_int64), ("dec_t_us", P), ("dec_m", P),
                ("dec_e", P), ("dec_B", P), ("dec_L_us", P), ("dec_score_q", P), ("dec_flags", P)]


class EsError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libedgeserve.so; raise loudly when it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EsError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        L.es_last_error.restype = ctypes.c_char_p
        L.es_version.restype = ctypes.c_char_p
        L.es_launch_count.restype = ctypes.c_int64
        L.es_launch_count.argtypes = [P]
        i32, u32, i64 = ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64
        sig = {
            "es_load_profile": [P, P, i32, i32, P],
            "es_free_profile": [P],
            "es_get_tables": [P, i32, P, P, P, P, i32, P, P],
            "es_score_candidates": [P, P, P, P],
            "es_replay_traces": [P, P, P, P],
            "es_scen_p95": [P, P, P, P],
            "es_scen_stats": [P, P, P, u32, P, P, P],
            "es_replay_traces_host": [P, P, P, P],
            "es_replay_traces_host_pipelined": [P, P, P, i32, P],
            "es_group_accumulate": [P, P, P, u32, P, P, P],
            "es_group_hist": [P, P, P, u32, i32, P, P, P],
            "es_group_p95_select": [u32, i32, P, P, P, P],
            "es_device_status": [P, P, P, P],
        }
        for f, args in sig.items():
            fn = getattr(L, f)
            fn.restype = ctypes.c_int
            fn.argtypes = args
        del i64
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise EsError(f"{STATUS.get(st, st)}: {lib().es_last_error().decode()}")


def _ptr(t):
    """data pointer of a torch tensor / numpy array / None."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(t, name):
    if t is not None and not t.is_cuda:
        raise EsError(f"{name} must be a CUDA tensor")


class Profile:
    """Library-owned profile handle (es_profile*)."""

    def __init__(self, handle, M, E, nb, cfgs, device):
        self.handle = handle
        self.M, self.E, self.nb = M, E, nb
        self.cfgs = cfgs
        self.device = device

    def __del__(self):
        try:
            if self.handle:
                lib().es_free_profile(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def launches(self):
        return int(lib().es_launch_count(self.handle))


def es_load_profile(profile, cfgs, device=0) -> Profile:
    """profile: inputs.Profile-like (M, E, bs, lat [M,E,nb], mask [M,E]);
    cfgs: sequence with tau, C, b_max, warmup."""
    bs = np.ascontiguousarray(profile.bs, np.int32)
    lat = np.ascontiguousarray(profile.lat, np.uint32)
    mask = None if profile.mask is None else np.ascontiguousarray(profile.mask, np.uint8)
    acc = getattr(profile, "acc", None)
    acc = None if acc is None else np.ascontiguousarray(acc, np.uint16)
    d = ProfileDesc(int(profile.M), int(profile.E), int(bs.size), bs.ctypes.data, lat.ctypes.data,
                    None if mask is None else mask.ctypes.data, None if acc is None else acc.ctypes.data)
    arr = (SchedCfg * len(cfgs))()
    for i, c in enumerate(cfgs):
        arr[i] = SchedCfg(int(c.tau), int(c.C), int(c.b_max), int(c.warmup), int(getattr(c, "policy", 0)))
    h = ctypes.c_void_p()
    _check(lib().es_load_profile(ctypes.byref(d), arr, len(cfgs), int(device), ctypes.byref(h)))
    return Profile(h, int(profile.M), int(profile.E), int(bs.size), list(cfgs), int(device))


def es_get_tables(prof: Profile, k: int):
    xc = ctypes.c_uint64()
    r = ctypes.c_uint32()
    nA = ctypes.c_int32()
    _check(lib().es_get_tables(prof.handle, k, ctypes.byref(xc), ctypes.byref(r), ctypes.byref(nA), None, 0,
                               None, None))
    A = np.zeros(nA.value, np.uint32)
    Bt = np.zeros(1024, np.uint32)
    H = np.zeros(prof.M * prof.E * prof.nb, np.uint64)
    _check(lib().es_get_tables(prof.handle, k, None, None, None, A.ctypes.data, nA.value, Bt.ctypes.data,
                               H.ctypes.data))
    return {"x_c": int(xc.value), "r": int(r.value), "A": A, "Bt": Bt, "H": H.reshape(prof.M, prof.E, prof.nb)}


def es_score_candidates(prof: Profile, q_off, waits, cfg_idx=None, cand=True, out=None, stream=None):
    """K1 on n snapshots.  q_off (u64 [n*M+1]) and waits (u32) are CUDA tensors."""
    import torch
    for t, nm in [(q_off, "q_off"), (waits, "waits"), (cfg_idx, "cfg_idx")]:
        _require_cuda(t, nm)
    n = (q_off.numel() - 1) // prof.M
    dev = q_off.device
    if out is None:
        out = {"m": torch.empty(n, dtype=torch.uint8, device=dev), "e": torch.empty(n, dtype=torch.uint8, device=dev),
               "B": torch.empty(n, dtype=torch.uint16, device=dev), "L": torch.empty(n, dtype=torch.uint32, device=dev),
               "S": torch.empty(n, dtype=torch.uint64, device=dev), "flags": torch.empty(n, dtype=torch.uint8, device=dev),
               "cand": torch.empty(n * prof.M, dtype=torch.uint64, device=dev) if cand else None}
    sn = Snapshots(n, _ptr(cfg_idx), _ptr(q_off), _ptr(waits), int(waits.numel()))
    dc = Decisions(_ptr(out["m"]), _ptr(out["e"]), _ptr(out["B"]), _ptr(out["L"]), _ptr(out["S"]),
                   _ptr(out["flags"]), _ptr(out.get("cand")))
    _check(lib().es_score_candidates(prof.handle, ctypes.byref(sn), ctypes.byref(dc), _stream(stream)))
    return out


def alloc_replay_out(prof: Profile, n_scen, total, device, full=True, p95=True, dec_cap=0):
    import torch
    o = {"latency": torch.empty(total, dtype=torch.uint32, device=device),
         "stats": torch.empty((n_scen, ES_NSTAT), dtype=torch.uint64, device=device),
         "p95": torch.empty(n_scen, dtype=torch.uint32, device=device) if p95 else None,
         "completion": torch.empty(total, dtype=torch.uint32, device=device) if full else None,
         "exit": torch.empty(total, dtype=torch.uint8, device=device) if full else None,
         "dec_cap": int(dec_cap)}
    if dec_cap:
        nd = n_scen * dec_cap
        for k, dt in [("dec_t", torch.uint32), ("dec_m", torch.uint8), ("dec_e", torch.uint8),
                      ("dec_B", torch.uint16), ("dec_L", torch.uint32), ("dec_S", torch.uint64),
                      ("dec_f", torch.uint8)]:
            o[k] = torch.zeros(nd, dtype=dt, device=device)
    return o


def _traces_struct(n_scen, arr_off, arrival, cfg_idx=None, group_id=None):
    return Traces(int(n_scen), _ptr(cfg_idx), _ptr(group_id), _ptr(arr_off), _ptr(arrival))


def _out_struct(o, p95=True):
    g = o.get
    return ReplayOut(_ptr(g("completion")), _ptr(g("exit")), _ptr(g("latency")), _ptr(g("stats")),
                     _ptr(g("p95")) if p95 else None, int(g("dec_cap") or 0), _ptr(g("dec_t")), _ptr(g("dec_m")),
                     _ptr(g("dec_e")), _ptr(g("dec_B")), _ptr(g("dec_L")), _ptr(g("dec_S")), _ptr(g("dec_f")))


def es_replay_traces(prof: Profile, arr_off, arrival, cfg_idx=None, group_id=None, out=None, full=True,
                     p95=True, dec_cap=0, stream=None):
    """K2 + K3 over every scenario.  Inputs are CUDA tensors (u64 arr_off
    [n*M+1], u32 arrival, optional u16 cfg_idx / u32 group_id)."""
    for t, nm in [(arr_off, "arr_off"), (arrival, "arrival"), (cfg_idx, "cfg_idx"), (group_id, "group_id")]:
        _require_cuda(t, nm)
    n = (arr_off.numel() - 1) // prof.M
    if out is None:
        out = alloc_replay_out(prof, n, arrival.numel(), arrival.device, full, p95, dec_cap)
    tr = _traces_struct(n, arr_off, arrival, cfg_idx, group_id)
    ro = _out_struct(out, p95)  # p95=False: K2 only (run K3 later with es_scen_p95)
    _check(lib().es_replay_traces(prof.handle, ctypes.byref(tr), ctypes.byref(ro), _stream(stream)))
    return out


def es_scen_p95(prof: Profile, arr_off, arrival, out, cfg_idx=None, stream=None):
    """K3 alone on the latencies a previous replay wrote into ``out``."""
    n = (arr_off.numel() - 1) // prof.M
    tr = _traces_struct(n, arr_off, arrival, cfg_idx, None)
    ro = _out_struct(out)
    _check(lib().es_scen_p95(prof.handle, ctypes.byref(tr), ctypes.byref(ro), _stream(stream)))
    return out


def es_scen_stats(prof: Profile, arr_off, arrival, out, n_groups=0, counts=None, hist0=None, cfg_idx=None,
                  group_id=None, p95=True, stream=None):
    """K3 fused with the level-0 group accumulation (one pass over latencies)."""
    n = (arr_off.numel() - 1) // prof.M
    tr = _traces_struct(n, arr_off, arrival, cfg_idx, group_id)
    ro = _out_struct(out, p95)
    _check(lib().es_scen_stats(prof.handle, ctypes.byref(tr), ctypes.byref(ro), ctypes.c_uint32(n_groups),
                               _ptr(counts), _ptr(hist0), _stream(stream)))
    return out


def es_replay_traces_host(prof: Profile, arr_off, arrival, cfg_idx=None, group_id=None, out=None,
                          stream=None):
    """End-to-end: host (ideally pinned) inputs and outputs; copies inside."""
    n = (arr_off.numel() - 1) // prof.M if hasattr(arr_off, "numel") else (arr_off.size - 1) // prof.M
    tr = _traces_struct(n, arr_off, arrival, cfg_idx, group_id)
    ro = _out_struct(out)
    _check(lib().es_replay_traces_host(prof.handle, ctypes.byref(tr), ctypes.byref(ro), _stream(stream)))
    return out


def es_replay_traces_host_pipelined(prof: Profile, batches, stream=None):
    """End-to-end over several host batches, each (arr_off, arrival, cfg_idx,
    group_id, out) with host (ideally pinned) arrays: the input copy of batch
    k+1 overlaps the replay of batch k.  Returns the list of outs."""
    nb = len(batches)
    trs = (Traces * nb)()
    ros = (ReplayOut * nb)()
    for i, (arr_off, arrival, cfg_idx, group_id, out) in enumerate(batches):
        n = (arr_off.numel() - 1) // prof.M if hasattr(arr_off, "numel") else (arr_off.size - 1) // prof.M
        trs[i] = _traces_struct(n, arr_off, arrival, cfg_idx, group_id)
        ros[i] = _out_struct(out)
    _check(lib().es_replay_traces_host_pipelined(prof.handle, trs, ros, ctypes.c_int32(nb), _stream(stream)))
    return [b[4] for b in batches]


def es_group_accumulate(prof, arr_off, arrival, out, n_groups, counts, hist0, cfg_idx=None, group_id=None,
                        stream=None):
    n = (arr_off.numel() - 1) // prof.M
    tr = _traces_struct(n, arr_off, arrival, cfg_idx, group_id)
    ro = _out_struct(out)
    _check(lib().es_group_accumulate(prof.handle, ctypes.byref(tr), ctypes.byref(ro), ctypes.c_uint32(n_groups),
                                     _ptr(counts), _ptr(hist0), _stream(stream)))


def es_group_hist(prof, arr_off, arrival, out, n_groups, level, state, hist, cfg_idx=None, group_id=None,
                  stream=None):
    n = (arr_off.numel() - 1) // prof.M
    tr = _traces_struct(n, arr_off, arrival, cfg_idx, group_id)
    ro = _out_struct(out)
    _check(lib().es_group_hist(prof.handle, ctypes.byref(tr), ctypes.byref(ro), ctypes.c_uint32(n_groups),
                               ctypes.c_int32(level), _ptr(state), _ptr(hist), _stream(stream)))


def es_group_p95_select(n_groups, level, counts, hist, state, stream=None):
    _check(lib().es_group_p95_select(ctypes.c_uint32(n_groups), ctypes.c_int32(level), _ptr(counts), _ptr(hist),
                                     _ptr(state), _stream(stream)))


def es_device_status(prof, stream=None):
    code = ctypes.c_uint32()
    item = ctypes.c_int64()
    _check(lib().es_device_status(prof.handle, _stream(stream), ctypes.byref(code), ctypes.byref(item)))
    return int(code.value), int(item.value)


from .engine import group_merge, replay_group_stats, upload_traces  # noqa: E402,F401
