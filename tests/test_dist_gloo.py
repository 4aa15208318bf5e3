"""Multi-rank plumbing on CPU (gloo, world_size 2): scenario sharding, the int64
all_reduce of u64 counters/histograms used between radix levels, and the exactness
of the group-P95 radix protocol of include/edgeserve.h (coarse min(T >> 12, 4095),
then T & 0xFFF, or T >> 20 / (T >> 8) & 0xFFF / T & 0xFF in overflow) after summing
per-rank histograms -- checked against the oracle's P95 of the union."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from paper_2605_05527_b200 import engine


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _digit(lat, level, ovf, prefix):
    """(take mask, bin) of one radix level, as documented in include/edgeserve.h."""
    if level == 0:
        return np.ones(lat.size, bool), np.minimum(lat >> 12, 4095)
    if not ovf:
        return (lat >> 12) == prefix, lat & 0xFFF
    big = (lat >> 12) >= 4095
    if level == 1:
        return big, lat >> 20
    if level == 2:
        return big & ((lat >> 20) == prefix), (lat >> 8) & 0xFFF
    return big & ((lat >> 8) == prefix), lat & 0xFF


def _hist_level(lat, level, ovf, prefix):
    take, b = _digit(lat, level, ovf, prefix)
    h = np.zeros(4096, np.uint64)
    np.add.at(h, b[take].astype(np.int64), 1)
    return h


def _select(h, rank_k):
    c = np.cumsum(h.astype(np.int64))
    b = int(np.searchsorted(c, rank_k))  # first bin with cumulative >= k
    before = int(c[b - 1]) if b else 0
    return b, rank_k - before


def _worker(rank, world, port, n_scen, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = engine.shard_ids(n_scen, rank, world)
    w = inputs.workload("cfg2", scen_ids=ids, n_req=600)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces)
    G = 13
    lats = [[] for _ in range(G)]
    counts = np.zeros((G, 2), np.uint64)  # completed, violations
    for s in range(w.traces.n_scen):
        g = int(w.traces.group_id[s])
        lo, hi = int(w.traces.arr_off[s * 4]), int(w.traces.arr_off[s * 4 + 4])
        lats[g].append(o["lat"][lo + 100:hi])
        counts[g] += o["stats"][s, [3, 4]]
    lats = [np.concatenate(x).astype(np.uint64) if x else np.zeros(0, np.uint64) for x in lats]
    ct = torch.from_numpy(counts.astype(np.int64))
    engine._all_reduce(ct, None)  # the product helper (int64 view of u64 sums)
    counts = ct.numpy().astype(np.uint64)
    result = []
    for g in range(G):
        N = int(counts[g, 0])
        k = (95 * N + 99) // 100
        prefix, ovf = 0, False
        for level in range(4):
            h = torch.from_numpy(_hist_level(lats[g], level, ovf, prefix).astype(np.int64))
            engine._all_reduce(h, None)
            if N == 0:
                continue
            b, k = _select(h.numpy(), k)
            if level == 0:
                prefix, ovf = b, b == 4095
            elif not ovf:
                prefix = (prefix << 12) | b
                break
            elif level == 1:
                prefix = b
            elif level == 2:
                prefix = (prefix << 12) | b
            else:
                prefix = (prefix << 8) | b
        result.append(prefix if N else 0)
    q.put((rank, ids.tolist(), counts.tolist(), result))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_two_rank_group_merge_is_exact():
    n_scen, world = 26, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_scen, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = sorted(sum((r[1] for r in res), []))
    assert ids == list(range(n_scen))  # shards partition the scenario set
    assert res[0][2] == res[1][2] and res[0][3] == res[1][3]  # every rank agrees
    w = inputs.workload("cfg2", scen_ids=np.arange(n_scen), n_req=600)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces)
    oc, op = oracle.group_stats(w.traces, o, w.cfgs, 13)
    assert [int(x) for x in op] == res[0][3]
    assert np.array_equal(np.array(res[0][2], np.uint64), oc[:, [3, 4]])


def test_shard_ids_partition():
    for n in [1, 7, 4096, 65536]:
        for world in [1, 2, 3, 8]:
            parts = [engine.shard_ids(n, r, world) for r in range(world)]
            assert np.array_equal(np.concatenate(parts), np.arange(n))
            assert max(p.size for p in parts) - min(p.size for p in parts) <= 1
