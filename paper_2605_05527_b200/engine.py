"""Host orchestration of the replay path and the per-group merge (step a10).

Everything numeric runs in libedgeserve.so; this module only moves tensors,
and (multi-GPU) calls torch.distributed.all_reduce(SUM) on the integer
counters and histograms between the three radix-selection levels of the group
P95.  Integer sums are order-independent, so the merged results are
bit-identical for any number of ranks.
"""
from __future__ import annotations

import numpy as np


def upload_traces(traces, device, pin=False):
    """inputs.Traces -> dict of CUDA tensors (u64 arr_off, u32 arrival, u16
    cfg_idx, u32 group_id)."""
    import torch

    def t(a, dt):
        x = torch.from_numpy(np.ascontiguousarray(a).view(dt_np[dt])).view(dt)
        if pin:
            x = x.pin_memory()
        return x.to(device, non_blocking=pin)

    dt_np = {torch.uint64: np.uint64, torch.uint32: np.uint32, torch.uint16: np.uint16}
    return {"arr_off": t(traces.arr_off, torch.uint64), "arrival": t(traces.arrival, torch.uint32),
            "cfg_idx": t(traces.cfg_idx, torch.uint16), "group_id": t(traces.group_id, torch.uint32)}


def _all_reduce(x, group):
    import torch
    import torch.distributed as dist
    if group is False or not dist.is_available() or not dist.is_initialized():
        return
    dist.all_reduce(x.view(torch.int64), op=dist.ReduceOp.SUM, group=group)


def group_merge(prof, dtr, out, n_groups, group=None, stream=None, with_p95=False, events=None):
    """Exact per-group counters and nearest-rank P95 across all ranks.

    dtr: uploaded traces of this rank's scenarios; out: this rank's replay
    outputs.  group: a torch.distributed process group (None = default when
    initialised, False = local only).  with_p95: also compute the per-scenario
    P95 (K3) in the same pass as the level-0 histogram.  Returns
    (counts u64 [G][ES_NGSTAT], p95 u64 [G]).
    """
    import torch
    from . import ES_HIST_BINS, ES_NGSTAT, es_group_hist, es_group_p95_select, es_scen_stats
    dev = dtr["arrival"].device
    G = int(n_groups)
    buf = torch.zeros(G * ES_NGSTAT + G * ES_HIST_BINS, dtype=torch.uint64, device=dev)
    counts = buf[:G * ES_NGSTAT]
    hist = buf[G * ES_NGSTAT:]
    state = torch.zeros(2 * G, dtype=torch.uint64, device=dev)
    es_scen_stats(prof, dtr["arr_off"], dtr["arrival"], out, G, counts, hist, dtr["cfg_idx"], dtr["group_id"],
                  p95=with_p95, stream=stream)
    if events:  # timing marks: after K3 + level 0, after the last level
        events[0].record(stream)
    _all_reduce(buf, group)
    es_group_p95_select(G, 0, counts, hist, state, stream)
    for level in (1, 2, 3):
        es_group_hist(prof, dtr["arr_off"], dtr["arrival"], out, G, level, state, hist, dtr["cfg_idx"],
                      dtr["group_id"], stream)
        _all_reduce(hist, group)
        es_group_p95_select(G, level, counts, hist, state, stream)
    if events:
        events[1].record(stream)
    return counts.view(G, ES_NGSTAT), state.view(G, 2)[:, 0]


def replay_group_stats(prof, dtr, n_groups, full=False, group=None, stream=None, out=None):
    """One pass of the whole hot path: K2 replay + K3 P95 + group merge."""
    from . import es_replay_traces
    out = es_replay_traces(prof, dtr["arr_off"], dtr["arrival"], dtr["cfg_idx"], dtr["group_id"], out=out,
                           full=full, p95=False, stream=stream)
    counts, p95 = group_merge(prof, dtr, out, n_groups, group=group, stream=stream, with_p95=True)
    return out, counts, p95


def shard_ids(n_total, rank, world):
    """Contiguous scenario block of `rank` when n_total scenarios are split over
    `world` ranks (strong scaling); the last ranks may get one fewer."""
    base, extra = divmod(int(n_total), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return np.arange(lo, hi, dtype=np.int64)


def weak_ids(per_rank, rank):
    """Weak scaling: rank r replays scenarios [r S, (r+1) S) of the config's sequence."""
    return np.arange(rank * per_rank, (rank + 1) * per_rank, dtype=np.int64)


# group-P95 radix levels (normal path): level 0 coarse min(T >> 12, 4095), level 1 T & 0xFFF
COARSE_SHIFT, COARSE_OVF = 12, 4095


def replay_group_stats_host(prof, host_batches, n_groups, group=None, stream=None):
    """End-to-end form of replay_group_stats over host batches (the call a user
    with traces in host memory makes).  host_batches: list of (hin, hout) with
    hin = {"arr_off", "arrival", "cfg_idx", "group_id"} pinned host tensors and
    hout = {"stats", "p95", "counts", "gp95"} pinned host tensors.  Per batch:
    the inputs go host -> device on a copy stream into one of two device
    buffers (batch k+1's copy overlaps batch k's replay), then K2 + K3 + the
    group merge (NCCL all_reduce across ranks when `group` is a process group)
    run on `stream`, and the per-scenario counters, per-scenario P95, group
    counters and group P95 come back device -> host.  Synchronises `stream`."""
    import torch
    from . import alloc_replay_out, es_replay_traces
    if not host_batches:
        return
    stream = stream or torch.cuda.current_stream()
    dev = stream.device
    hin0 = host_batches[0][0]
    bufs = [{k: torch.empty_like(v, device=dev) for k, v in hin0.items()} for _ in range(2)]
    n = (hin0["arr_off"].numel() - 1) // prof.M
    out = alloc_replay_out(prof, n, hin0["arrival"].numel(), dev, full=False, p95=True)
    copy = torch.cuda.Stream(device=dev)
    ev_copied = [torch.cuda.Event(), torch.cuda.Event()]
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]
    copy.wait_stream(stream)
    for k, (hin, hout) in enumerate(host_batches):
        b = k & 1
        d = bufs[b]
        assert all(hin[x].shape == hin0[x].shape for x in hin0), "equal batch shapes"
        with torch.cuda.stream(copy):
            if k >= 2:
                copy.wait_event(ev_done[b])
            for x in d:
                d[x].copy_(hin[x], non_blocking=True)
            ev_copied[b].record(copy)
        stream.wait_event(ev_copied[b])
        with torch.cuda.stream(stream):
            es_replay_traces(prof, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], out=out, full=False,
                             p95=False, stream=stream)
            counts, gp95 = group_merge(prof, d, out, n_groups, group=group, stream=stream, with_p95=True)
            hout["stats"].copy_(out["stats"], non_blocking=True)
            hout["p95"].copy_(out["p95"], non_blocking=True)
            hout["counts"].copy_(counts, non_blocking=True)
            hout["gp95"].copy_(gp95, non_blocking=True)
            ev_done[b].record(stream)
    stream.synchronize()
