"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit-exact.

Every comparison is element by element on the same seeded inputs (inputs/):
tables, per-snapshot decisions and candidate scores (K1), per-request
completion / exit / latency, decision logs and per-scenario counters (K2),
per-scenario P95 (K3) and merged group statistics (a10).
"""
import numpy as np
import pytest

import inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2605_05527_b200 as es  # noqa: E402

DEV = "cuda:0"


def np_of(t):
    return t.cpu().numpy() if t is not None else None


def to_dev(a, dt):
    m = {torch.uint64: np.uint64, torch.uint32: np.uint32, torch.uint16: np.uint16, torch.uint8: np.uint8}
    return torch.from_numpy(np.ascontiguousarray(a).astype(m[dt])).to(DEV)


# ------------------------------------------------------------------ tables

@pytest.mark.parametrize("C", [1, 2, 10, 15])
def test_tables_bitwise(C):
    taus = [1024, 1500, 20000, 25000, 33333, 50000, 70001, 100000, 1 << 20]
    prof = inputs.synth_profile(4, 4, list(range(1, 17)))
    cfgs = [inputs.SchedCfg(tau=t, b_max=16, C=C) for t in taus]
    # the image must fit shared memory: split the large-tau cfg out
    for chunk in (cfgs[:-1], cfgs[-1:]):
        h = es.es_load_profile(prof, chunk)
        for k, c in enumerate(chunk):
            g = es.es_get_tables(h, k)
            o = oracle.build_tables(c.tau, C)
            assert g["x_c"] == o["x_c"] and g["r"] == o["r"]
            assert np.array_equal(g["A"], o["A"]), (c.tau, C)
            assert np.array_equal(g["Bt"], o["Bt"])
            for m in range(4):
                for e in range(4):
                    for b in range(16):
                        L = int(prof.lat[m, e, b])
                        exp = oracle.H(c.tau, L)[0] if L < o["x_c"] else np.iinfo(np.uint64).max
                        assert int(g["H"][m, e, b]) == exp


def test_profile_validation_errors():
    p = inputs.synth_profile(3, 3, [1, 2, 4, 8])
    bad = p.lat.copy()
    bad[2, 1, 3] = bad[2, 0, 3]
    with pytest.raises(es.EsError, match="MONOTONE.*m=2,e=1,b=3"):
        es.es_load_profile(inputs.Profile(3, 3, p.bs, bad, p.mask), [inputs.SchedCfg(50000, 8)])
    with pytest.raises(es.EsError, match="OUT_OF_GRID"):
        es.es_load_profile(p, [inputs.SchedCfg(50000, 9)])
    with pytest.raises(es.EsError, match="ARG"):
        es.es_load_profile(p, [inputs.SchedCfg(500, 8)])
    with pytest.raises(es.EsError, match="GRID"):
        es.es_load_profile(inputs.Profile(3, 3, np.array([2, 4, 6, 8], np.int32), p.lat, p.mask),
                           [inputs.SchedCfg(50000, 8)])


# ------------------------------------------------------------------ K1

def run_k1(prof, cfgs, q_off, waits, cfg_idx=None):
    h = es.es_load_profile(prof, cfgs)
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(waits, torch.uint32),
                               None if cfg_idx is None else to_dev(cfg_idx, torch.uint16))
    torch.cuda.synchronize()
    return {k: np_of(v) for k, v in o.items()}


def assert_k1_equal(g, o, M):
    for k in ["m", "e", "B", "L", "S", "flags"]:
        assert np.array_equal(g[k], o[k]), (k, np.nonzero(g[k] != o[k])[0][:10])
    assert np.array_equal(g["cand"].reshape(-1, M), o["cand"])


@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 8])
def test_k1_random_states(M):
    """SPEC-style random states: queues <= 10, waits in [0, 3 tau]."""
    prof = inputs.synth_profile(M, 4, list(range(1, 11)), L_top=28000.0)
    cfgs = [inputs.SchedCfg(tau=50000, b_max=10), inputs.SchedCfg(tau=20000, b_max=7)]
    n = 3000
    q_off, w = inputs.snapshots_uniform(40 + M, n, M, 10, 150000)
    ci = (np.arange(n) % 2).astype(np.uint16)
    assert_k1_equal(run_k1(prof, cfgs, q_off, w, ci), oracle.decide_batch(prof, cfgs, q_off, w, ci), M)


@pytest.mark.parametrize("M,depth", [(4, 300), (8, 4096)])
def test_k1_deep_snapshots(M, depth):
    """5-C-style deep queues: long clipped prefixes counted, not read."""
    prof = inputs.synth_profile(M, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
    rate = inputs.rates_for_shallow_load(prof, 32, 1.5)
    q_off, w = inputs.snapshots_poisson_depth(7, np.arange(160), M, depth, rate)
    assert_k1_equal(run_k1(prof, cfgs, q_off, w), oracle.decide_batch(prof, cfgs, q_off, w), M)


@pytest.mark.parametrize("base_off", [0, 1, 3])
def test_k1_stream_live_windows(monkeypatch, base_off):
    """The streaming mapping on all-live deep queues (the HBM regime of the
    bench): warp ranges cut queues at arbitrary positions, the waits pointer is
    misaligned by base_off elements (scalar heads/tails around the 16-byte
    body), B* up to 64 (served heads longer than a warp), two SLOs, a few
    clip-path snapshots mixed in, and inversions planted in bodies, at 16-byte
    boundaries and in the last wait of a queue (flagged bad, Q24)."""
    monkeypatch.setenv("ES_K1", "stream")
    M = 8
    prof = inputs.synth_profile(M, 5, list(range(1, 65)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=64), inputs.SchedCfg(tau=80000, b_max=40)]
    n = 600
    q_off, w = inputs.snapshots_poisson_depth(11, np.arange(n), M, 1500, [1500 / 100000.0] * M)
    w = w.copy()
    rng = np.random.default_rng(5)
    # clip path: push the head of a few snapshots near x_c
    clip = rng.choice(n, 20, replace=False)
    for s in clip:
        lo, hi = int(q_off[s * M]), int(q_off[s * M + 1])
        if hi > lo:
            w[lo] = max(int(w[lo]), 170000)
    # inversions: body, 16-byte boundary, last wait of a queue
    planted = []
    for s in rng.choice(np.setdiff1d(np.arange(n), clip), 12, replace=False):
        m = int(rng.integers(M))
        lo, hi = int(q_off[s * M + m]), int(q_off[s * M + m + 1])
        if hi - lo < 10:
            continue
        pos = [lo + (hi - lo) // 2, (lo + 5) & ~3, hi - 1][len(planted) % 3]
        pos = min(max(pos, lo + 1), hi - 1)
        w[pos] = w[pos - 1] + 1
        planted.append(s)
    ci = (np.arange(n) % 2).astype(np.uint16)
    h = es.es_load_profile(prof, cfgs)
    buf = np.zeros(w.size + base_off, np.uint32)
    buf[base_off:] = w
    dw = to_dev(buf, torch.uint32)[base_off:]
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), dw, to_dev(ci, torch.uint16))
    torch.cuda.synchronize()
    g = {k: np_of(v) for k, v in o.items()}
    ref = oracle.decide_batch(prof, cfgs, q_off, w, ci)
    assert_k1_equal(g, ref, M)
    assert (ref["flags"][planted] & 4).all()  # every planted inversion is in the read window


@pytest.mark.parametrize("base_off", [0, 1, 3])
def test_k1_thread_balanced_pass(monkeypatch, base_off):
    """The thread-per-snapshot mapping's balanced pass (one SLO per warp, the
    region of 32 snapshots' waits cut into shared-memory chunks of `cap`
    positions): regions far above one chunk (queues up to 60 over 8 models),
    a waits pointer misaligned by base_off elements, empty queues, a batch
    size that is not a multiple of 32, a few clip-path snapshots (handed to the
    warp segments), a warp with two SLOs (the per-lane loop), and inversions
    planted inside queues, at their last wait and at a chunk-sized stride
    (flagged bad, Q24) -- element by element against the oracle."""
    monkeypatch.setenv("ES_K1", "thread")
    M = 8
    prof = inputs.synth_profile(M, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32), inputs.SchedCfg(tau=90000, b_max=20)]
    n = 32 * 23 + 7
    q_off, w = inputs.snapshots_uniform(77, n, M, 60, 60000)
    w = w.copy()
    rng = np.random.default_rng(9)
    ci = np.zeros(n, np.uint16)
    ci[32 * 3:32 * 4] = 1          # a whole warp on the second SLO (balanced pass, its tables)
    ci[32 * 5 + 7] = 1             # one warp with two SLOs (per-lane loop)
    clip = rng.choice(n, 6, replace=False)
    for s in clip:  # clip path: a head past x_c - max L
        lo, hi = int(q_off[s * M]), int(q_off[s * M + 1])
        if hi > lo:
            w[lo] = 200000
    planted = []
    for j, s in enumerate(rng.choice(np.setdiff1d(np.arange(n), clip), 14, replace=False)):
        m = int(rng.integers(M))
        lo, hi = int(q_off[s * M + m]), int(q_off[s * M + m + 1])
        if hi - lo < 3:
            continue
        pos = [lo + (hi - lo) // 2, hi - 1][j % 2]
        w[pos] = w[pos - 1] + 1
        planted.append(s)
    h = es.es_load_profile(prof, cfgs)
    buf = np.zeros(w.size + base_off, np.uint32)
    buf[base_off:] = w
    dw = to_dev(buf, torch.uint32)[base_off:]
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), dw, to_dev(ci, torch.uint16))
    torch.cuda.synchronize()
    g = {k: np_of(v) for k, v in o.items()}
    ref = oracle.decide_batch(prof, cfgs, q_off, w, ci)
    assert_k1_equal(g, ref, M)
    assert (ref["flags"][planted] & 4).all()
    assert (ref["flags"] & 4).sum() >= len(planted)


def test_k1_masks_and_flags():
    """exit masks (ablation), no-work, bad input, bad cfg index."""
    prof = inputs.synth_profile(3, 4, [1, 2, 4, 8])
    prof.mask = np.array([[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 0, 1]], np.uint8)
    cfgs = [inputs.SchedCfg(tau=30000, b_max=8)]
    q_off, w = inputs.snapshots_uniform(5, 800, 3, 9, 80000)
    assert_k1_equal(run_k1(prof, cfgs, q_off, w), oracle.decide_batch(prof, cfgs, q_off, w), 3)
    # no work + an inversion in the live window + a cfg index out of range
    q = np.array([0, 0, 0, 0, 2, 3, 3, 4, 5, 6], np.uint64)
    ws = np.array([10, 20, 7, 9, 8, 7], np.uint32)
    g = run_k1(prof, cfgs, q, ws, np.array([0, 0, 5], np.uint16))
    assert list(g["flags"]) == [2, 4, 4]


def test_k1_harvested_snapshots():
    """Snapshots harvested from oracle replays of cfg2/cfg3 traces."""
    for name, ids in [("cfg2", [1, 7]), ("cfg3", [2, 11])]:
        w = inputs.workload(name, scen_ids=ids, n_req=1500)
        M = w.profile.M
        cap = 3000
        o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap)
        q_off, ws, ci = inputs.harvest_snapshots(w.traces, o["stats"][:, 0], cap, o["dec_t"], o["dec_m"], o["dec_B"])
        g = run_k1(w.profile, w.cfgs, q_off, ws, ci)
        r = oracle.decide_batch(w.profile, w.cfgs, q_off, ws, ci)
        assert_k1_equal(g, r, M)


# ------------------------------------------------------------------ K2 / K3

def run_k2(w, full=True, dec_cap=0):
    h = es.es_load_profile(w.profile, w.cfgs)
    d = es.upload_traces(w.traces, DEV)
    out = es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], full=full,
                              dec_cap=dec_cap)
    torch.cuda.synchronize()
    code, item = es.es_device_status(h)
    res = {k: (np_of(v) if hasattr(v, "cpu") else v) for k, v in out.items()}
    res["_handle"], res["_dev"], res["_out"] = h, d, out
    res["_code"] = code
    return res


def assert_k2_equal(g, o, dec_cap=0):
    assert np.array_equal(g["stats"], o["stats"]), np.nonzero((g["stats"] != o["stats"]).any(1))[0][:10]
    assert np.array_equal(g["p95"], o["p95"])
    if "completion" in o and g.get("completion") is not None:
        assert np.array_equal(g["completion"], o["completion"])
        assert np.array_equal(g["exit"], o["exit"])
        assert np.array_equal(g["latency"], o["lat"])
    if dec_cap:
        for k in ["dec_t", "dec_m", "dec_e", "dec_B", "dec_L", "dec_S", "dec_f"]:
            assert np.array_equal(g[k], o[k]), k


@pytest.mark.parametrize("name,ids,n_req", [
    ("cfg1", [0], None),
    ("cfg2", list(range(0, 130, 3)), 2500),
    ("cfg3", list(range(0, 117, 5)), 2000),
])
def test_k2_parity_configs(name, ids, n_req):
    w = inputs.workload(name, scen_ids=ids, n_req=n_req)
    cap = 4000
    g = run_k2(w, dec_cap=cap)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap, nthreads=8)
    assert g["_code"] == 0
    assert_k2_equal(g, o, cap)


def test_k2_deep_overload():
    """5-B-shaped overload (rho_shallow 1.5): deep queues, clipped prefixes."""
    w = inputs.workload("cfg5b", scen_ids=[0, 1, 2], n_req=12000)
    g = run_k2(w)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, nthreads=3)
    assert int(o["stats"][:, 6].max()) > 500  # really deep
    assert_k2_equal(g, o)


def test_k2_edge_cases():
    prof = inputs.synth_profile(3, 3, [1, 2, 4, 8])
    cfgs = [inputs.SchedCfg(tau=50000, b_max=8, warmup=0), inputs.SchedCfg(tau=20000, b_max=3, warmup=2)]
    scen = [
        [[], [], []],                      # empty scenario
        [[0], [], []],                     # single request
        [[5] * 40, [5] * 3, [5]],          # everything at one instant (Q10)
        [[], [], list(range(0, 100000, 7))],  # one busy model only
        [[10, 10, 4000000000], [], []],    # long idle gap (Q12)
        [[1, 2, 3], [7, 8], []],
    ]
    segs = [[np.asarray(q, np.uint32) for q in sc] for sc in scen]
    n = len(scen)
    tr = inputs._assemble(3, segs, [i % 2 for i in range(n)], [0] * n, np.arange(n))
    w = inputs.Workload("edge", prof, cfgs, tr, 0)
    g = run_k2(w, dec_cap=64)
    o = oracle.replay_batch(prof, cfgs, tr, dec_cap=64)
    assert_k2_equal(g, o, 64)


def test_k2_errors():
    prof = inputs.synth_profile(2, 2, [1, 2])
    cfgs = [inputs.SchedCfg(tau=50000, b_max=2, warmup=0)]
    scen = [[[5, 3], []], [[0xFFFFFFF0], [1]], [[1], [2]]]  # unsorted, u32 overflow, fine
    segs = [[np.asarray(q, np.uint32) for q in sc] for sc in scen]
    tr = inputs._assemble(2, segs, [0, 0, 0], [0] * 3, np.arange(3))
    w = inputs.Workload("err", prof, cfgs, tr, 0)
    g = run_k2(w)
    o = oracle.replay_batch(prof, cfgs, tr)
    assert int(g["stats"][0, 7]) == 8 and int(o["stats"][0, 7]) != 0  # ES_ERR_UNSORTED
    assert int(g["stats"][1, 7]) == 5 and int(o["stats"][1, 7]) == 3  # ES_ERR_RANGE / oracle RANGE
    assert np.array_equal(g["stats"][2], o["stats"][2])
    assert g["_code"] in (5, 8)


def test_group_merge_matches_oracle():
    w = inputs.workload("cfg2", scen_ids=np.arange(52), n_req=1500)
    g = run_k2(w)
    counts, p95 = es.group_merge(g["_handle"], g["_dev"], g["_out"], 13, group=False)
    torch.cuda.synchronize()
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, nthreads=8)
    oc, op = oracle.group_stats(w.traces, o, w.cfgs, 13)
    assert np.array_equal(np_of(counts), oc)
    assert np.array_equal(np_of(p95).astype(np.uint32), op)


def test_host_entry_point_matches_device():
    w = inputs.workload("cfg2", scen_ids=np.arange(20), n_req=1200)
    h = es.es_load_profile(w.profile, w.cfgs)
    tr = w.traces
    total = tr.arrival.size
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    ho = {"latency": pin(np.zeros(total, np.uint32)), "stats": pin(np.zeros((tr.n_scen, es.ES_NSTAT), np.uint64)),
          "p95": pin(np.zeros(tr.n_scen, np.uint32)), "completion": pin(np.zeros(total, np.uint32)),
          "exit": pin(np.zeros(total, np.uint8)), "dec_cap": 0}
    es.es_replay_traces_host(h, pin(tr.arr_off), pin(tr.arrival), pin(tr.cfg_idx), pin(tr.group_id), out=ho)
    o = oracle.replay_batch(w.profile, w.cfgs, tr, nthreads=4)
    g = {k: (v.numpy() if hasattr(v, "numpy") else v) for k, v in ho.items()}
    assert_k2_equal(g, o)


def test_host_pipelined_batches_match_oracle():
    """es_replay_traces_host_pipelined: five batches of different sizes and
    configs through the double-buffered pipeline (input copy of batch k+1
    overlapping the replay of batch k); every batch equals the oracle."""
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    w0 = inputs.workload("cfg2", scen_ids=np.arange(3), n_req=500)
    h = es.es_load_profile(w0.profile, w0.cfgs)
    batches, refs = [], []
    for k, ids in enumerate([np.arange(20), np.arange(40, 47), np.arange(100, 160), np.arange(5), np.arange(7, 30)]):
        w = inputs.workload("cfg2", scen_ids=ids, n_req=800 + 200 * k)
        tr = w.traces
        total = tr.arrival.size
        ho = {"latency": pin(np.zeros(total, np.uint32)), "stats": pin(np.zeros((tr.n_scen, es.ES_NSTAT), np.uint64)),
              "p95": pin(np.zeros(tr.n_scen, np.uint32)), "completion": pin(np.zeros(total, np.uint32)),
              "exit": pin(np.zeros(total, np.uint8)), "dec_cap": 0}
        batches.append((pin(tr.arr_off), pin(tr.arrival), pin(tr.cfg_idx), pin(tr.group_id), ho))
        refs.append(oracle.replay_batch(w.profile, w.cfgs, tr, nthreads=4))
    es.es_replay_traces_host_pipelined(h, batches)
    for (_, _, _, _, ho), o in zip(batches, refs):
        assert_k2_equal({k: (v.numpy() if hasattr(v, "numpy") else v) for k, v in ho.items()}, o)


def test_full_size_cfg2_bench_config():
    """BASELINE configs[1] at full size in the bench's launch configuration:
    every scenario's counters and P95 against the oracle (16 host threads),
    plus full per-request outputs on a sample of scenarios."""
    w = inputs.workload("cfg2")
    g = run_k2(w, full=False)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, full=True, nthreads=16)
    assert np.array_equal(g["stats"], o["stats"])
    assert np.array_equal(g["p95"], o["p95"])
    assert np.array_equal(g["latency"], o["lat"])
    counts, p95 = es.group_merge(g["_handle"], g["_dev"], g["_out"], 13, group=False)
    oc, op = oracle.group_stats(w.traces, o, w.cfgs, 13)
    assert np.array_equal(np_of(counts), oc) and np.array_equal(np_of(p95).astype(np.uint32), op)


def test_determinism_repeat():
    w = inputs.workload("cfg3", scen_ids=np.arange(40), n_req=800)
    a = run_k2(w)
    b = run_k2(w)
    for k in ["stats", "p95", "completion", "exit", "latency"]:
        assert np.array_equal(a[k], b[k])


def test_group_merge_rank_count_invariance():
    """Split the scenarios over W = 1, 2, 4, 8 emulated ranks on one GPU: each
    shard replays and histograms its own scenarios; the per-shard u64 buffers
    are summed (what all_reduce(sum) does) between the radix levels.  Counters
    and P95 must be bit-identical for every W and equal the oracle's."""
    from paper_2605_05527_b200 import engine
    n, G = 40, 13
    w = inputs.workload("cfg2", scen_ids=np.arange(n), n_req=900)
    h = es.es_load_profile(w.profile, w.cfgs)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, nthreads=8)
    oc, op = oracle.group_stats(w.traces, o, w.cfgs, G)
    results = []
    for W in (1, 2, 4, 8):
        shards = []
        for r in range(W):
            sub = inputs.workload("cfg2", scen_ids=engine.shard_ids(n, r, W), n_req=900)
            d = es.upload_traces(sub.traces, DEV)
            out = es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], full=False)
            shards.append((d, out))
        bufs = []
        for d, out in shards:
            buf = torch.zeros(G * es.ES_NGSTAT + G * 4096, dtype=torch.uint64, device=DEV)
            es.es_group_accumulate(h, d["arr_off"], d["arrival"], out, G, buf[:G * es.ES_NGSTAT], buf[G * es.ES_NGSTAT:], d["cfg_idx"],
                                   d["group_id"])
            bufs.append(buf)
        tot = bufs[0].view(torch.int64).clone()
        for b in bufs[1:]:
            tot += b.view(torch.int64)
        tot = tot.view(torch.uint64)
        counts, hist = tot[:G * es.ES_NGSTAT], tot[G * es.ES_NGSTAT:]
        state = torch.zeros(2 * G, dtype=torch.uint64, device=DEV)
        es.es_group_p95_select(G, 0, counts, hist, state)
        for level in (1, 2):
            acc = torch.zeros(G * 4096, dtype=torch.int64, device=DEV)
            for d, out in shards:
                hl = torch.empty(G * 4096, dtype=torch.uint64, device=DEV)
                es.es_group_hist(h, d["arr_off"], d["arrival"], out, G, level, state, hl, d["cfg_idx"], d["group_id"])
                acc += hl.view(torch.int64)
            es.es_group_p95_select(G, level, counts, acc.view(torch.uint64), state)
        torch.cuda.synchronize()
        results.append((np_of(counts).reshape(G, es.ES_NGSTAT), np_of(state).reshape(G, 2)[:, 0]))
    for c, p in results:
        assert np.array_equal(c, oc)
        assert np.array_equal(p.astype(np.uint32), op)


def test_group_merge_overflow_bin():
    """Group P95 beyond 16.77 s (the coarse overflow bin): the 4-level path."""
    prof = inputs.Profile(M=1, E=1, bs=np.array([1], np.int32), lat=np.array([[[12000]]], np.uint32),
                          mask=np.ones((1, 1), np.uint8))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=1, warmup=5)]
    scen = [[[0] * 1900], [list(range(0, 3000000, 7000))], [[10] * 1500 + [20000000] * 30]]
    segs = [[np.asarray(q, np.uint32) for q in sc] for sc in scen]
    tr = inputs._assemble(1, segs, [0, 0, 0], [0, 1, 0], np.arange(3))
    w = inputs.Workload("ovf", prof, cfgs, tr, 0)
    g = run_k2(w)
    counts, p95 = es.group_merge(g["_handle"], g["_dev"], g["_out"], 2, group=False, with_p95=False)
    torch.cuda.synchronize()
    o = oracle.replay_batch(prof, cfgs, tr)
    oc, op = oracle.group_stats(tr, o, cfgs, 2)
    assert int(op[0]) > (4095 << 12)  # really in the overflow bin
    assert np.array_equal(np_of(counts), oc)
    assert np.array_equal(np_of(p95).astype(np.uint32), op)
    assert np.array_equal(g["p95"], o["p95"])


@pytest.mark.parametrize("lps", ["8", "16", "32"])
def test_k2_segment_widths(monkeypatch, lps):
    """Every K2 segment width (ES_LPS = 8, 16, 32 lanes per scenario) gives the
    oracle's bits on config subsets, deep overload (the general clip path),
    the edge cases and the errors."""
    monkeypatch.setenv("ES_LPS", lps)
    for name, ids, n_req in [("cfg1", [0], None), ("cfg2", list(range(0, 60, 3)), 1500),
                             ("cfg3", list(range(0, 117, 2)), 1500)]:
        w = inputs.workload(name, scen_ids=ids, n_req=n_req)
        g = run_k2(w, dec_cap=2000)
        o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=2000, nthreads=8)
        assert g["_code"] == 0
        assert_k2_equal(g, o, 2000)
    test_k2_deep_overload()
    test_k2_edge_cases()
    test_k2_errors()


@pytest.mark.parametrize("M", [1, 3, 5])
def test_k1_thread_balanced_pass_small_m(monkeypatch, M):
    """The balanced pass with fewer models than the template width (M < 8, 4,
    2: queues past M absent), one SLO and no cfg index array, regions over
    several chunks, empty queues and a ragged batch, against the oracle."""
    monkeypatch.setenv("ES_K1", "thread")
    prof = inputs.synth_profile(M, 4, list(range(1, 17)))
    cfgs = [inputs.SchedCfg(tau=60000, b_max=16)]
    n = 32 * 11 + 13
    q_off, w = inputs.snapshots_uniform(90 + M, n, M, 90, 80000)
    h = es.es_load_profile(prof, cfgs)
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(w, torch.uint32))
    torch.cuda.synchronize()
    assert_k1_equal({k: np_of(v) for k, v in o.items()}, oracle.decide_batch(prof, cfgs, q_off, w), M)


@pytest.mark.parametrize("mode", ["stream", "thread", "seg"])
def test_k1_all_mappings(monkeypatch, mode):
    """K1's mappings (3-phase streaming and one CTA per snapshot for deep
    queues, warp segments for small ones) on every K1 input family."""
    monkeypatch.setenv("ES_K1", mode)
    test_k1_random_states(3)
    test_k1_random_states(8)
    test_k1_deep_snapshots(8, 4096)
    test_k1_deep_snapshots(4, 300)
    test_k1_masks_and_flags()
    test_k1_harvested_snapshots()


def test_k1_full_size_bench_batch():
    """K1 at the bench's full size and launch configuration (bench.k1_batch:
    262,144 5-C snapshots, 17.3 GB of waits, the TMA stream mapping): 512
    sampled snapshots spread over every tile against the oracle, element by
    element, plus properties that hold for every snapshot (Eq. 7's choice is
    the argmin of the candidate scores, Q3 tie-break)."""
    import bench
    q_off, w0, tiles = bench.k1_batch(0)
    M = 8
    n = (q_off.size - 1) // M
    prof = inputs.synth_profile(8, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
    h = es.es_load_profile(prof, cfgs)
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(w0, torch.uint32).repeat(tiles))
    torch.cuda.synchronize()
    g = {k: np_of(v) for k, v in o.items()}
    # sampled snapshots: their queues re-packed into a small CSR for the oracle
    rng = np.random.default_rng(3)
    ids = np.sort(rng.choice(n, 512, replace=False))
    n0 = n // tiles
    sub_off, parts = [0], []
    for s in ids:
        s0 = s % n0  # tile copies share the seeded waits of snapshot s0
        for m in range(M):
            lo, hi = int(q_off[s0 * M + m]), int(q_off[s0 * M + m + 1])
            parts.append(w0[lo:hi])
            sub_off.append(sub_off[-1] + hi - lo)
    ref = oracle.decide_batch(prof, cfgs, np.array(sub_off, np.uint64), np.concatenate(parts))
    sub = {k: g[k][ids] for k in ["m", "e", "B", "L", "S", "flags"]}
    sub["cand"] = g["cand"].reshape(-1, M)[ids]
    assert_k1_equal(sub, ref, M)
    # every snapshot: the chosen model is the (S, m) argmin of its candidate scores
    cand = g["cand"].reshape(-1, M)
    ok = g["flags"] & 6 == 0
    assert np.array_equal(np.argmin(cand[ok], axis=1), g["m"][ok].astype(np.int64))
    assert np.array_equal(cand[ok].min(axis=1), g["S"][ok])


def _tiled_sample_parity(prof, cfgs, q_off, w0, ci, tiles, n_sample, seed):
    """bench.k1_line's launch on the distinct snapshots (q_off, w0, ci) repeated
    `tiles` times back to back, then n_sample snapshots spread over every tile
    against the oracle element by element (their queues re-packed into a small
    CSR), plus the argmin property on every snapshot."""
    M = prof.M
    n0 = (q_off.size - 1) // M
    nw = np.uint64(w0.size)
    q = np.concatenate([q_off[:-1] + np.uint64(t) * nw for t in range(tiles)] + [q_off[-1:] + np.uint64(tiles - 1) * nw])
    h = es.es_load_profile(prof, cfgs)
    dci = None if ci is None else to_dev(np.tile(ci, tiles), torch.uint16)
    o = es.es_score_candidates(h, to_dev(q, torch.uint64), to_dev(w0, torch.uint32).repeat(tiles), dci)
    torch.cuda.synchronize()
    g = {k: np_of(v) for k, v in o.items()}
    rng = np.random.default_rng(seed)
    ids = np.sort(rng.choice(n0 * tiles, n_sample, replace=False))
    sub_off, parts = [0], []
    for s in ids:
        s0 = s % n0
        for m in range(M):
            lo, hi = int(q_off[s0 * M + m]), int(q_off[s0 * M + m + 1])
            parts.append(w0[lo:hi])
            sub_off.append(sub_off[-1] + hi - lo)
    sub_ci = None if ci is None else ci[ids % n0]
    ref = oracle.decide_batch(prof, cfgs, np.array(sub_off, np.uint64), np.concatenate(parts), sub_ci)
    sub = {k: g[k][ids] for k in ["m", "e", "B", "L", "S", "flags"]}
    sub["cand"] = g["cand"].reshape(-1, M)[ids]
    assert_k1_equal(sub, ref, M)
    cand = g["cand"].reshape(-1, M)
    ok = g["flags"] & 6 == 0
    assert np.array_equal(np.argmin(cand[ok], axis=1), g["m"][ok].astype(np.int64))
    assert np.array_equal(cand[ok].min(axis=1), g["S"][ok])
    return g


def test_k1_clip_bench_batch():
    """K1 at the bench's `k1_clip` size and launch (bench.bench_k1_clip: 5-C
    depth at 5-B overload rates, 262,144 snapshots, every one on the clip path:
    k1s_prep + k1s_clip + k1s_finish): 256 sampled snapshots against the oracle."""
    prof = inputs.synth_profile(8, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
    rate = inputs.rates_for_shallow_load(prof, 32, 1.5)
    q_off, w0 = inputs.snapshots_poisson_depth(2000, np.arange(4096), 8, 4096, rate)
    g = _tiled_sample_parity(prof, cfgs, q_off, w0, None, 64, 256, 5)
    assert (g["flags"] & 1).sum() == 0  # overload: nothing feasible, as in the bench line


def test_k1_harvested_bench_batch():
    """K1 at the bench's `k1_harvested` size and launch (bench.k1_harvested_batch:
    every decision instant of 512 cfg3 replays, nine SLOs, 8 tiles, the
    thread-per-snapshot mapping): 512 sampled snapshots against the oracle."""
    import bench
    from paper_2605_05527_b200 import engine
    dev = torch.device(DEV)
    _, q_off, w0, ci, _ = bench.k1_harvested_batch(es, engine, dev, torch.cuda.current_stream(dev), 0, 512)
    w = inputs.workload("cfg3", scen_ids=[0], n_req=10)
    _tiled_sample_parity(w.profile, w.cfgs, q_off, w0, ci, 8, 512, 6)


# ------------------------------------------------------------------ baseline / ablation policies (Q26)

POLICY_IDS = {"edgeserving": 0, "all_final": 1, "all_early": 2, "ee_lqf": 3, "ee_edf": 4, "allfinal_da": 5,
              "ours_bs1": 6, "symphony": 7, "grid": 8}


def with_policies(w, pols):
    """The workload with one cfg per policy (same SLO knobs as cfg 0) and
    scenario s on policy pols[s % len(pols)] -- segments of one warp mix
    policies."""
    import dataclasses
    c0 = w.cfgs[0]
    cfgs = [inputs.SchedCfg(tau=c0.tau, b_max=c0.b_max, C=c0.C, warmup=c0.warmup, policy=POLICY_IDS[p])
            for p in pols]
    ci = (np.arange(w.traces.n_scen) % len(pols)).astype(np.uint16)
    return dataclasses.replace(w, cfgs=cfgs, traces=dataclasses.replace(w.traces, cfg_idx=ci))


@pytest.mark.parametrize("policy", list(POLICY_IDS))
def test_k2_policy_parity(policy):
    """Every policy alone (cfg2 shape, 4 models x 4 exits, LPS 16; cfg3 shape,
    8 models x 5 exits, LPS 32, bursty MMPP): completions, exits, latencies,
    decision logs, counters and P95 bit-exact against the oracle."""
    cap = 3000
    for name, ids, n_req in [("cfg2", list(range(0, 60, 3)), 2000), ("cfg3", list(range(0, 45, 5)), 1500)]:
        w = with_policies(inputs.workload(name, scen_ids=ids, n_req=n_req), [policy])
        g = run_k2(w, dec_cap=cap)
        o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap, nthreads=8)
        assert g["_code"] == 0
        assert_k2_equal(g, o, cap)


def test_k2_mixed_policies_in_one_warp():
    """All nine policies interleaved scenario by scenario (every warp mixes
    scoring and LQF / EDF segments)."""
    cap = 3000
    w = with_policies(inputs.workload("cfg2", scen_ids=list(range(70)), n_req=1500), list(POLICY_IDS))
    g = run_k2(w, dec_cap=cap)
    o = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=cap, nthreads=8)
    assert g["_code"] == 0
    assert_k2_equal(g, o, cap)


def test_k1_rejects_deferred_batching():
    """es_score_candidates scores every policy but SYMPHONY (its wait-until
    needs a replay clock; include/edgeserve.h)."""
    prof = inputs.synth_profile(2, 2, [1, 2])
    h = es.es_load_profile(prof, [inputs.SchedCfg(tau=50000, b_max=2, policy=7)])
    q_off, w = inputs.snapshots_uniform(1, 4, 2, 3, 100000)
    with pytest.raises(es.EsError):
        es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(w, torch.uint32))


@pytest.mark.parametrize("M", [3, 8])
def test_k1_policies(M):
    """K1 under the baseline / ablation policies and GRID (Q26, Q28), one cfg
    per policy interleaved snapshot by snapshot: decisions, scores (per-model
    best cell under GRID, none under LQF / EDF) and flags equal the oracle,
    with inversions planted in some snapshots (flagged bad, Q24)."""
    pols = [p for p in POLICY_IDS if p != "symphony"]
    prof = inputs.synth_profile(M, 4, [1, 2, 4, 8], L_top=20000.0)
    cfgs = [inputs.SchedCfg(tau=50000, b_max=6, policy=POLICY_IDS[p]) for p in pols]
    n = 1800
    q_off, w = inputs.snapshots_uniform(60 + M, n, M, 9, 150000)
    w = w.copy()
    rng = np.random.default_rng(M)
    for s in rng.choice(n, 40, replace=False):
        m = int(rng.integers(M))
        lo, hi = int(q_off[s * M + m]), int(q_off[s * M + m + 1])
        if hi - lo >= 2:
            w[hi - 1] = w[hi - 2] + 1
    ci = (np.arange(n) % len(pols)).astype(np.uint16)
    assert_k1_equal(run_k1(prof, cfgs, q_off, w, ci), oracle.decide_batch(prof, cfgs, q_off, w, ci), M)


@pytest.mark.parametrize("mode", ["thread", "seg", "stream"])
def test_many_slos_core_staging(monkeypatch, mode):
    """24 SLO cfgs (tau 20..135 ms) on the 8 x 5 x 32 profile: the whole image
    (~390 KB) exceeds shared memory, so every kernel stages the core and reads
    H from global memory -- K1 on every mapping and K2, against the oracle."""
    monkeypatch.setenv("ES_K1", mode)
    prof = inputs.synth_profile(8, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=20000 + 5000 * k, b_max=32) for k in range(24)]
    M, n = 8, 200
    depth = 1500 if mode == "stream" else 40
    q_off, wts = inputs.snapshots_poisson_depth(31, np.arange(n), M, depth, [depth / 90000.0] * M)
    ci = (np.arange(n) % 24).astype(np.uint16)
    h = es.es_load_profile(prof, cfgs)
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(wts, torch.uint32), to_dev(ci, torch.uint16))
    torch.cuda.synchronize()
    assert_k1_equal({k: np_of(v) for k, v in o.items()}, oracle.decide_batch(prof, cfgs, q_off, wts, ci), M)
    if mode == "thread":  # K2 replay under the same 24 cfgs (cfg3-shaped traces, cfg index s mod 24)
        w = inputs.workload("cfg3", scen_ids=list(range(0, 96, 4)), n_req=1200)
        tr = w.traces
        tr.cfg_idx = (np.arange(tr.n_scen) % 24).astype(np.uint16)
        w2 = inputs.Workload("slo24", prof, cfgs, tr, 0)
        g = run_k2(w2, dec_cap=1500)
        ref = oracle.replay_batch(prof, cfgs, tr, dec_cap=1500, nthreads=8)
        assert g["_code"] == 0
        assert_k2_equal(g, ref, 1500)


@pytest.mark.parametrize("fast", ["tma", "regs"])
def test_k1_stream_large_image(monkeypatch, fast):
    """Deep snapshots under cfg3's nine SLOs (20..100 ms): the profile image
    is ~145 KB, so the TMA ring drops to 2 KB pieces x 2 slots (and the
    register-pipelined kernel is the ES_K1_FAST=regs variant); per-snapshot
    SLO index, mixed fast / clip-path snapshots (short SLOs clip)."""
    monkeypatch.setenv("ES_K1", "stream")
    monkeypatch.setenv("ES_K1_FAST", fast)
    w = inputs.workload("cfg3", scen_ids=[0], n_req=10)
    M = 8
    n = 270
    q_off, wts = inputs.snapshots_poisson_depth(21, np.arange(n), M, 1600, [1600 / 90000.0] * M)
    ci = (np.arange(n) % 9).astype(np.uint16)
    h = es.es_load_profile(w.profile, w.cfgs)
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(wts, torch.uint32), to_dev(ci, torch.uint16))
    torch.cuda.synchronize()
    g = {k: np_of(v) for k, v in o.items()}
    ref = oracle.decide_batch(w.profile, w.cfgs, q_off, wts, ci)
    assert_k1_equal(g, ref, M)


def test_k1_stream_extreme_shapes(monkeypatch):
    """The TMA streaming mapping on its edge shapes: one snapshot with a single
    3M-wait queue (every warp range inside one queue, no boundary) and 20,000
    snapshots of 0-3 waits per queue (several queue and snapshot boundaries
    in every 128-wait window, empty queues and empty snapshots)."""
    monkeypatch.setenv("ES_K1", "stream")
    M = 8
    prof = inputs.synth_profile(M, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
    h = es.es_load_profile(prof, cfgs)
    # one deep queue: waits non-increasing, all live (< fast_lim)
    n_big = 3_000_000
    w = (np.arange(n_big, 0, -1, dtype=np.int64) * 120000 // n_big).astype(np.uint32)
    q_off = np.zeros(M + 1, np.uint64)
    q_off[3:] = n_big
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(w, torch.uint32))
    torch.cuda.synchronize()
    assert_k1_equal({k: np_of(v) for k, v in o.items()}, oracle.decide_batch(prof, cfgs, q_off, w), M)
    # many tiny snapshots
    q_off, w = inputs.snapshots_uniform(77, 20000, M, 3, 100000)
    o = es.es_score_candidates(h, to_dev(q_off, torch.uint64), to_dev(w, torch.uint32))
    torch.cuda.synchronize()
    assert_k1_equal({k: np_of(v) for k, v in o.items()}, oracle.decide_batch(prof, cfgs, q_off, w), M)


def test_k2_launch_shape_invariance(monkeypatch):
    """The scenario hand-out order (longest span first vs index order), the CTA
    size and the image staging (full vs core-only with H from global) change
    where and when scenarios run, never their results."""
    w = inputs.workload("cfg3", scen_ids=list(range(0, 90, 4)), n_req=1200)  # nine SLOs: 145 KB image
    ref = oracle.replay_batch(w.profile, w.cfgs, w.traces, dec_cap=2000, nthreads=8)
    for env in [{}, {"ES_K2_ORDER": "0"}, {"ES_K2_BLOCK": "64"}, {"ES_K2_BLOCK": "256", "ES_K2_ORDER": "0"}]:
        for k in ["ES_K2_ORDER", "ES_K2_BLOCK"]:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        g = run_k2(w, dec_cap=2000)
        assert g["_code"] == 0
        assert_k2_equal(g, ref, 2000)


# ------------------------------------------------------------------ round-2 parity gaps

@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
@pytest.mark.parametrize("exits", ["layer1+final", "layer3+final"])
def test_k2_restricted_exit_masks(name, exits):
    """K2 replay under the exit configurations of the paper's exit-point study
    (the f3 sweep): only {layer1, final} or {layer3, final} allowed
    for every model.  Eq. 6 searches the allowed exits only, the Q2 fallback is
    the shallowest *allowed* exit, cells count allowed exits; compared element
    by element (completions, exits, latencies, decision logs, counters)."""
    w = inputs.workload(name, scen_ids=list(range(0, 117, 4)), n_req=1500)
    E = w.profile.E
    keep = [0, E - 1] if exits == "layer1+final" else [2, E - 1]
    mask = np.zeros((w.profile.M, E), np.uint8)
    mask[:, keep] = 1
    prof = inputs.Profile(w.profile.M, E, w.profile.bs, w.profile.lat, mask, w.profile.acc)
    w = inputs.Workload(w.name, prof, w.cfgs, w.traces, w.n_req)
    g = run_k2(w, dec_cap=1500)
    o = oracle.replay_batch(prof, w.cfgs, w.traces, dec_cap=1500, nthreads=8)
    assert g["_code"] == 0
    nd = np.minimum(o["stats"][:, 0], 1500).astype(np.int64)
    valid = np.arange(1500)[None, :] < nd[:, None]
    assert set(np.unique(o["dec_e"].reshape(-1, 1500)[valid])) <= set(keep)
    assert_k2_equal(g, o, 1500)
    # cells examined = decisions' non-empty queues x 2 allowed exits
    assert np.array_equal(g["stats"][:, 2], 2 * g["stats"][:, 1])


@pytest.mark.parametrize("mode", ["seg", "stream", "block"])
def test_k1_q24_clipped_prefix_contract(monkeypatch, mode):
    """Reading Q24 exactly: K1 counts the clipped prefix (waits >= x_c) by
    search and never reads it, so an inversion planted *inside* that prefix is
    not flagged: the kernel returns the decision of the same snapshot with the
    prefix sorted, without ES_FLAG_BAD_INPUT, while the oracle (which checks
    whole queues) flags it.  Its neighbours in the batch are unaffected."""
    monkeypatch.setenv("ES_K1", mode)
    M = 4
    prof = inputs.synth_profile(M, 4, list(range(1, 17)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=16)]
    x_c = oracle.build_tables(50000, 10)["x_c"]
    depth = 1500 if mode != "seg" else 24
    q_off, w = inputs.snapshots_poisson_depth(3, np.arange(64), M, depth, [depth / 100000.0] * M)
    w = w.copy()
    lens = np.diff(q_off.astype(np.int64)).reshape(64, M)
    targets = [s for s in range(3, 64, 7) if lens[s, s % M] >= 6][:3]
    assert len(targets) == 3
    fixed = w.copy()
    for s in targets:
        m = s % M
        lo, hi = int(q_off[s * M + m]), int(q_off[s * M + m + 1])
        # a clipped prefix of 4 tasks (w >= x_c) with an inversion between its
        # 2nd and 3rd task; the rest of the queue stays below x_c
        pre = np.array([x_c + 5000, x_c + 3000, x_c + 9000, x_c + 100], np.uint32)
        w[lo:lo + 4] = pre
        fixed[lo:lo + 4] = np.sort(pre)[::-1]
        w[lo + 4:hi] = np.minimum(w[lo + 4:hi], x_c - 1)
        fixed[lo + 4:hi] = w[lo + 4:hi]
    g = run_k1(prof, cfgs, q_off, w)
    ref_bad = oracle.decide_batch(prof, cfgs, q_off, w)
    ref_fix = oracle.decide_batch(prof, cfgs, q_off, fixed)
    assert (ref_bad["flags"][targets] & 4).all()  # the oracle checks whole queues
    assert not (g["flags"][targets] & 4).any()  # the kernel does not read the prefix
    for k in ["m", "e", "B", "L", "S", "flags"]:
        assert np.array_equal(g[k], ref_fix[k]), k  # = the decision with the prefix sorted, every snapshot
    others = np.setdiff1d(np.arange(64), targets)
    assert np.array_equal(g["flags"][others], ref_bad["flags"][others])
    assert len(targets) == 3


def test_group_select_ranks_past_2_32():
    """The group P95 radix selection keeps the residual rank as a full u64:
    synthetic histograms with 6e9 and 5e9 completions (far past 2^32), one
    resolved at level 1, one through the overflow levels 1-3."""
    G, B = 2, es.ES_HIST_BINS
    counts = torch.zeros(G * es.ES_NGSTAT, dtype=torch.uint64, device=DEV)
    c = np.zeros((G, es.ES_NGSTAT), np.int64)
    c[0, 3], c[1, 3] = 6_000_000_000, 5_000_000_000
    counts.copy_(torch.from_numpy(c.reshape(-1)).view(torch.uint64))
    state = torch.zeros(2 * G, dtype=torch.uint64, device=DEV)

    def hist(entries):
        h = np.zeros((G, B), np.int64)
        for g, b, v in entries:
            h[g, b] = v
        return torch.from_numpy(h.reshape(-1)).view(torch.uint64).to(DEV)

    # level 0: group 0 rank ceil(0.95*6e9)=5.7e9 -> coarse bin 20 (after 5e9 in bin 10), residual 0.7e9;
    # group 1: everything in the overflow bin 4095, rank 4.75e9
    es.es_group_p95_select(G, 0, counts, hist([(0, 10, 5_000_000_000), (0, 20, 1_000_000_000),
                                              (1, 4095, 5_000_000_000)]), state)
    # level 1: group 0 T & 0xFFF inside bin 20 -> residual 0.7e9 lands in bin 9 (after 0.5e9 in bin 7);
    # group 1 T >> 20: 3e9 in bin 20, 2e9 in bin 30 -> bin 30, residual 1.75e9
    es.es_group_p95_select(G, 1, counts, hist([(0, 7, 500_000_000), (0, 9, 500_000_000),
                                              (1, 20, 3_000_000_000), (1, 30, 2_000_000_000)]), state)
    # level 2 (overflow only): (T >> 8) & 0xFFF: bin 5 1e9, bin 6 1e9 -> bin 6, residual 0.75e9
    es.es_group_p95_select(G, 2, counts, hist([(1, 5, 1_000_000_000), (1, 6, 1_000_000_000)]), state)
    # level 3: T & 0xFF: bin 100 0.75e9, bin 200 1.25e9 -> bin 100
    es.es_group_p95_select(G, 3, counts, hist([(1, 100, 750_000_000), (1, 200, 1_250_000_000)]), state)
    torch.cuda.synchronize()
    p95 = np_of(state.view(G, 2)[:, 0]).astype(np.int64)
    assert int(p95[0]) == (20 << 12) | 9
    assert int(p95[1]) == (((30 << 12) | 6) << 8) | 100


def test_k2_golden_work_counters(monkeypatch):
    """The hand-computed replays of tests/golden/work_counters.json through the
    GPU replay (every segment width): counters, latencies and P95."""
    from test_oracle_counters import GOLD, expected_row, golden_case
    for lps in ["8", "16", "32"]:
        monkeypatch.setenv("ES_LPS", lps)
        for case in GOLD["cases"]:
            prof, cfgs, tr = golden_case(case)
            g = run_k2(inputs.Workload("golden", prof, cfgs, tr, 0))
            assert np.array_equal(g["stats"][0], expected_row(case)), (lps, case["name"], g["stats"][0])
            assert np.array_equal(g["latency"], np.asarray(case["latency"], np.uint32))
            assert int(g["p95"][0]) == case["p95"]


def test_full_size_cfg3_bench_config_sampled():
    """BASELINE configs[2] (the bench headline) at full size -- 65,536 scenarios
    x 8 DNNs x 5 exits x batch 1-32, MMPP, 9 SLOs -- in the bench's launch
    configuration (the segment width the library picks for this batch): 512
    scenarios spread over the batch are replayed one by one by the oracle and
    compared element by element (counters, P95, every latency); the group
    merge is checked against the per-scenario counters it sums (all 117
    groups) and its P95 against the nearest-rank definition (Q15) applied to
    the replayed latencies of three whole groups."""
    w = inputs.workload("cfg3")
    g = run_k2(w, full=False)
    assert g["_code"] == 0
    S = w.traces.n_scen
    ids = np.unique(np.linspace(0, S - 1, 512).astype(np.int64))
    sub = inputs.workload("cfg3", scen_ids=ids)
    o = oracle.replay_batch(sub.profile, sub.cfgs, sub.traces, full=True, nthreads=16)
    assert np.array_equal(g["stats"][ids], o["stats"])
    assert np.array_equal(g["p95"][ids], o["p95"])
    off = w.traces.arr_off
    for j, s in enumerate(ids):
        a, b = int(off[s * 8]), int(off[s * 8 + 8])
        so = sub.traces.arr_off
        assert np.array_equal(g["latency"][a:b], o["lat"][int(so[j * 8]):int(so[j * 8 + 8])]), s
    G = inputs.n_groups("cfg3")
    counts, p95 = es.group_merge(g["_handle"], g["_dev"], g["_out"], G, group=False)
    cols = oracle.GROUP_SRC
    ref = np.zeros((G, len(cols)), np.uint64)
    np.add.at(ref, w.traces.group_id.astype(np.int64), g["stats"][:, cols])
    assert np.array_equal(np_of(counts), ref)
    p95 = np_of(p95)
    for grp in [0, 58, 116]:
        vals = []
        for s in np.nonzero(w.traces.group_id == grp)[0]:
            W = w.cfgs[int(w.traces.cfg_idx[s])].warmup
            vals.append(g["latency"][int(off[s * 8]) + W:int(off[s * 8 + 8])])
        v = np.sort(np.concatenate(vals))
        k = (95 * v.size + 99) // 100
        assert int(p95[grp]) == int(v[k - 1]), grp



def test_k3_ragged_sizes_and_value_ranges():
    """K3 alone (es_scen_p95) on synthetic latency segments: every size class
    around the 16-byte quads and the CTA width (0 .. 30,001 post-warmup values,
    base offsets at every alignment), value ranges that take the per-lane coarse
    bins (< 131 ms), the shared coarse bins (131 ms .. 16.77 s), the overflow
    radix select (>= 16.77 s), ties and zeros -- against the oracle's nearest-rank
    P95 (reading Q15) of the post-warmup values."""
    import torch
    prof = inputs.Profile(M=1, E=1, bs=np.array([1], np.int32), lat=np.array([[[1000]]], np.uint32),
                          mask=np.ones((1, 1), np.uint8))
    W = 5
    h = es.es_load_profile(prof, [inputs.SchedCfg(tau=50000, b_max=1, warmup=W)])
    rng = np.random.default_rng(2605)
    sizes = [0, 3, 5, 6, 7, 8, 9, 10, 12, 13, 36, 38, 261, 262, 1028, 1030, 4104, 12292, 12296, 30006]
    kinds = ["small", "wide", "ties", "huge", "zeros", "edge"]
    segs = []
    for i, n in enumerate(sizes * len(kinds)):
        kind = kinds[i // len(sizes)]
        if kind == "small":
            v = rng.integers(0, 131_000, n)
        elif kind == "wide":
            v = rng.integers(0, 16_000_000, n)
        elif kind == "ties":
            v = np.full(n, 40_960)
        elif kind == "huge":
            v = np.where(rng.random(n) < 0.2, rng.integers(0, 50_000, n), rng.integers(16_777_216, 2**32 - 1, n))
        elif kind == "zeros":
            v = np.zeros(n, np.int64)
        else:  # values on the coarse-bin edges (multiples of 4096 and one below)
            v = rng.integers(0, 40, n) * 4096 - rng.integers(0, 2, n)
            v = np.maximum(v, 0)
        segs.append(np.asarray(v, np.uint32))
    arr_off = np.zeros(len(segs) + 1, np.uint64)
    arr_off[1:] = np.cumsum([s.size for s in segs])
    lat = np.concatenate(segs).astype(np.uint32)
    dev = "cuda:0"
    out = {"latency": torch.from_numpy(lat.view(np.int32)).to(dev).view(torch.uint32),
           "stats": torch.zeros((len(segs), es.ES_NSTAT), dtype=torch.uint64, device=dev),
           "p95": torch.full((len(segs),), 0xFFFFFFFF, dtype=torch.uint32, device=dev),
           "dec_cap": 0}
    d_off = torch.from_numpy(arr_off.view(np.int64)).to(dev).view(torch.uint64)
    d_arr = torch.zeros(max(1, lat.size), dtype=torch.uint32, device=dev)
    es.es_scen_p95(h, d_off, d_arr, out)
    torch.cuda.synchronize()
    got = np_of(out["p95"])
    for i, s in enumerate(segs):
        want = oracle.p95(s[W:]) if s.size > W else 0
        assert int(got[i]) == want, (i, s.size, kinds[i // len(sizes)])
