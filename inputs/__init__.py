"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no urgency, score, batch or
exit rule, no replay).  It only produces *data*: latency profiles, request
traces and queue snapshots, with the shapes of the paper's workloads
(§VI-A) and the north-star configs (BASELINE.json).
Every random number comes from a counter-based splitmix64 stream keyed by
(seed, scenario, model, stream), so any subset of scenarios can be generated
independently (sampling at full size, sharding across ranks) and the result is
bit-identical wherever it is generated.

Recipes:
  * profile  L(m,e,b) = floor(L_top * kappa^((m-(M-1))/(M-1))
                               * delta^((e-(E-1))/(E-1)) * (1 + g (b-1)) + 1/2)
             L_top=12000 us, kappa=2, delta=7, g=(ratio-1)/(B_max-1), ratio=2.5
             (Fig. profile_mean laws: batch 1->B_max 2-3x, final
             6-8x layer1, heavier models slower).
  * rates    lambda_m proportional to (M - m) (3:2:1 for M=3), scaled so
             rho_full = sum_m lambda_m L(m, deepest, B_max) / B_max hits the target.
  * Poisson  per model, i.i.d. exponential gaps by inverse CDF, accumulated in
             float64, arrival = floor(cumulative), kept while < D where
             D = n_req / sum(lambda).
  * MMPP     one 2-state modulating chain per scenario shared by all models:
             burst x3 (mean sojourn 100 ms), calm x0.5 (400 ms), pi_burst=0.2
             (mean rate preserved); arrivals by time change of a unit-rate
             Poisson stream through the integrated intensity.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# stream tags (keep distinct)
STREAM_ARRIVAL = 1
STREAM_MMPP = 2
STREAM_SNAPSHOT = 3
STREAM_DEPTH = 4


def splitmix64(x):
    """Vectorised splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def stream_key(seed, scen, model, stream):
    """Key of the counter stream for (seed, scenario, model, stream tag)."""
    scen = np.asarray(scen, dtype=np.uint64)
    with np.errstate(over="ignore"):
        k = splitmix64(np.uint64(seed) ^ splitmix64(np.uint64(stream) * np.uint64(1 << 40) + np.uint64(model)))
        return splitmix64(k ^ splitmix64(scen * np.uint64(0x100000001B3) + np.uint64(7)))


def uniform01(keys, n):
    """uniform [0,1) doubles, shape keys.shape + (n,): u_k = top53(splitmix(key + (k+1) GOLD))."""
    keys = np.asarray(keys, dtype=np.uint64)[..., None]
    ctr = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = splitmix64(keys + ctr * _GOLD)
    return (x >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# --------------------------------------------------------------------------- profile


@dataclass
class Profile:
    """Latency table L(m, e, b) in integer microseconds."""

    M: int
    E: int
    bs: np.ndarray  # int32 [nb], strictly increasing, bs[0] == 1
    lat: np.ndarray  # uint32 [M, E, nb]
    mask: np.ndarray  # uint8 [M, E]
    acc: np.ndarray = None  # uint16 [M, E] top-1 accuracy, basis points (Table I), or None

    @property
    def nb(self) -> int:
        return int(self.bs.shape[0])


def synth_profile(M, E, bs, b_max=None, L_top=12000.0, kappa=2.0, delta=7.0, ratio=2.5,
                  mask=None) -> Profile:
    bs = np.asarray(bs, dtype=np.int32)
    if b_max is None:
        b_max = int(bs[-1])
    g = (ratio - 1.0) / (b_max - 1) if b_max > 1 else 0.0
    lat = np.zeros((M, E, len(bs)), dtype=np.uint32)
    for m in range(M):
        fm = kappa ** ((m - (M - 1)) / (M - 1)) if M > 1 else 1.0
        for e in range(E):
            fe = delta ** ((e - (E - 1)) / (E - 1)) if E > 1 else 1.0
            for i, b in enumerate(bs):
                lat[m, e, i] = math.floor(L_top * fm * fe * (1.0 + g * (int(b) - 1)) + 0.5)
    if mask is None:
        mask = np.ones((M, E), dtype=np.uint8)
    return Profile(M=M, E=E, bs=bs, lat=lat, mask=np.asarray(mask, dtype=np.uint8), acc=synth_accuracy(M, E))


# Table I: top-1 accuracy (%) on CIFAR-100 of ResNet50/101/152 at
# layer1, layer2, layer3, final -- in basis points (0.01 %)
TABLE_I_BP = np.array([[760, 1210, 3080, 7440], [740, 1450, 5430, 7790], [730, 1720, 4740, 7800]], np.int64)


def synth_accuracy(M, E):
    """Accuracy table shaped by Table I: model m takes the row of ResNet
    (3 m) // M (lighter models first, as the latency profile orders them);
    E = 4 uses the row as printed, other E interpolate it linearly at the exit
    fractions e / (E - 1) over the four exits at 0, 1/3, 2/3, 1.  Data only."""
    out = np.zeros((M, E), np.uint16)
    xs = np.array([0.0, 1 / 3, 2 / 3, 1.0])
    for m in range(M):
        row = TABLE_I_BP[(3 * m) // M]
        for e in range(E):
            x = e / (E - 1) if E > 1 else 1.0
            out[m, e] = row[e] if E == 4 else int(round(float(np.interp(x, xs, row.astype(np.float64)))))
    return out


def batch_index_of(bs, b_max):
    """Index of the largest profiled batch size <= b_max (input-shaping helper)."""
    return int(np.searchsorted(np.asarray(bs), b_max, side="right") - 1)


def rates_for_load(prof: Profile, b_max: int, rho: float):
    """lambda_m in requests/us, lambda_m ∝ (M - m), scaled to rho_full."""
    M = prof.M
    w = np.array([M - m for m in range(M)], dtype=np.float64)
    bi = batch_index_of(prof.bs, b_max)
    cost = np.array([prof.lat[m, prof.E - 1, bi] / b_max for m in range(M)], dtype=np.float64)
    scale = rho / float((w * cost).sum())
    return w * scale


def rates_for_shallow_load(prof: Profile, b_max: int, rho: float):
    """Overload variant (5-B): rho_shallow uses the shallowest exit."""
    M = prof.M
    w = np.array([M - m for m in range(M)], dtype=np.float64)
    bi = batch_index_of(prof.bs, b_max)
    cost = np.array([prof.lat[m, 0, bi] / b_max for m in range(M)], dtype=np.float64)
    return w * (rho / float((w * cost).sum()))


# --------------------------------------------------------------------------- traces


@dataclass
class SchedCfg:
    tau: int  # SLO deadline, us
    b_max: int
    C: int = 10
    warmup: int = 100
    policy: int = 0  # selection rule id (C ABI ES_POLICY_*): 0 = EdgeServing, 1..6 = paper baselines/ablations


@dataclass
class Traces:
    """CSR of (scenario, model) arrival segments, u32 us, sorted per segment."""

    M: int
    arr_off: np.ndarray  # uint64 [n_scen*M + 1]
    arrival: np.ndarray  # uint32 [total]
    cfg_idx: np.ndarray  # uint16 [n_scen]
    group_id: np.ndarray  # uint32 [n_scen]
    scen_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))

    @property
    def n_scen(self) -> int:
        return int(self.cfg_idx.shape[0])

    def scenario(self, s):
        """arrival arrays per model for local scenario s."""
        return [self.arrival[self.arr_off[s * self.M + m]:self.arr_off[s * self.M + m + 1]]
                for m in range(self.M)]


def _assemble(M, per_scen_lists, cfg_idx, group_id, scen_ids):
    counts = np.array([[len(x) for x in lst] for lst in per_scen_lists], dtype=np.uint64).reshape(-1)
    arr_off = np.zeros(counts.size + 1, dtype=np.uint64)
    np.cumsum(counts, out=arr_off[1:])
    parts = [x for lst in per_scen_lists for x in lst]
    arrival = np.concatenate(parts).astype(np.uint32) if parts else np.zeros(0, np.uint32)
    return Traces(M=M, arr_off=arr_off, arrival=arrival, cfg_idx=np.asarray(cfg_idx, np.uint16),
                  group_id=np.asarray(group_id, np.uint32), scen_ids=np.asarray(scen_ids, np.int64))


def _unit_gaps_cum(keys, K):
    """cumulative sums of K unit-rate exponential gaps per key (float64, sequential)."""
    u = uniform01(keys, K)
    gaps = -np.log1p(-u)
    return np.cumsum(gaps, axis=-1)


def poisson_segments(seed, scen_ids, lam, D, block=256):
    """Per scenario list of per-model u32 arrival arrays.

    lam: float64 [n, M] rates per us; D: float64 [n] durations in us.
    """
    scen_ids = np.asarray(scen_ids, dtype=np.int64)
    n, M = lam.shape
    if n and float(np.max(D)) >= 2.0 ** 32:
        raise ValueError("trace duration exceeds u32 microseconds (71.6 min)")
    out = [[None] * M for _ in range(n)]
    for b0 in range(0, n, block):
        b1 = min(n, b0 + block)
        ids = scen_ids[b0:b1]
        for m in range(M):
            mu = lam[b0:b1, m] * D[b0:b1]
            K = int(math.ceil(float(mu.max()) + 8.0 * math.sqrt(float(mu.max())) + 16))
            keys = stream_key(seed, ids, m, STREAM_ARRIVAL)
            cum = _unit_gaps_cum(keys, K) / lam[b0:b1, m][:, None]
            for j in range(b1 - b0):
                row = cum[j]
                cnt = int(np.searchsorted(row, D[b0 + j], side="left"))
                if cnt >= K:
                    raise RuntimeError("poisson generator margin exhausted")
                out[b0 + j][m] = np.floor(row[:cnt]).astype(np.uint32)
    return out


def mmpp_segments(seed, scen_ids, lam, D, burst=3.0, calm=0.5, soj_burst=100000.0,
                  soj_calm=400000.0, pi_burst=0.2):
    """Bursty MMPP arrivals (north star 'bursty MMPP')."""
    scen_ids = np.asarray(scen_ids, dtype=np.int64)
    n, M = lam.shape
    out = [[None] * M for _ in range(n)]
    for j in range(n):
        sid = scen_ids[j]
        # modulating chain: initial state, then alternating exponential sojourns
        nseg = int(D[j] / (soj_burst + soj_calm) * 2 + 64)
        key = stream_key(seed, sid, 0, STREAM_MMPP)
        u = uniform01(key, 2 * nseg + 1)
        state = 1 if u[0] < pi_burst else 0
        bounds = [0.0]
        rates = []
        k = 1
        while bounds[-1] < D[j]:
            if k >= u.size:
                u = np.concatenate([u, uniform01(splitmix64(key + np.uint64(k)), 2 * nseg)])
            mean = soj_burst if state else soj_calm
            bounds.append(bounds[-1] - mean * math.log1p(-float(u[k])))
            rates.append(burst if state else calm)
            state ^= 1
            k += 1
        bounds = np.asarray(bounds)
        rates = np.asarray(rates)
        Lam = np.concatenate([[0.0], np.cumsum(np.diff(bounds) * rates)])  # Λ at bounds
        LamD = float(np.interp(D[j], bounds, Lam))
        for m in range(M):
            mu = lam[j, m] * LamD
            K = int(math.ceil(mu + 8.0 * math.sqrt(mu) + 16))
            y = _unit_gaps_cum(stream_key(seed, sid, m + 1, STREAM_MMPP), K) / lam[j, m]
            cnt = int(np.searchsorted(y, LamD, side="left"))
            if cnt >= K:
                raise RuntimeError("mmpp generator margin exhausted")
            y = y[:cnt]
            seg = np.clip(np.searchsorted(Lam, y, side="right") - 1, 0, rates.size - 1)
            t = bounds[seg] + (y - Lam[seg]) / rates[seg]
            out[j][m] = np.floor(t).astype(np.uint32)
    return out


# --------------------------------------------------------------------------- snapshots


def snapshots_uniform(seed, n, M, max_len, w_max, len_lo=0):
    """SPEC-style random states: per queue length U[len_lo, max_len],
    waits U[0, w_max] integer us, sorted head-first (non-increasing)."""
    ids = np.arange(n, dtype=np.int64)
    lens = np.zeros((n, M), dtype=np.int64)
    lu = uniform01(stream_key(seed, ids, 0, STREAM_DEPTH), M)
    lens[:] = len_lo + np.floor(lu * (max_len - len_lo + 1)).astype(np.int64)
    q_off = np.zeros(n * M + 1, dtype=np.uint64)
    np.cumsum(lens.reshape(-1), out=q_off[1:])
    waits = np.zeros(int(q_off[-1]), dtype=np.uint32)
    for s in range(n):
        for m in range(M):
            k = int(lens[s, m])
            if k == 0:
                continue
            u = uniform01(stream_key(seed, s, m, STREAM_SNAPSHOT), k)
            w = np.floor(u * (w_max + 1)).astype(np.uint32)
            waits[q_off[s * M + m]:q_off[s * M + m + 1]] = np.sort(w)[::-1]
    return q_off, waits


def snapshots_poisson_depth(seed, scen_ids, M, depth_max, rate_per_us):
    """5-C style deep snapshots: per-model depth U[0, depth_max]; waits are
    floor(t - Poisson arrivals) in FIFO order (head = oldest = largest wait)."""
    scen_ids = np.asarray(scen_ids, dtype=np.int64)
    n = scen_ids.size
    lu = uniform01(stream_key(seed, scen_ids, 0, STREAM_DEPTH), M)
    lens = np.floor(lu * (depth_max + 1)).astype(np.int64)
    q_off = np.zeros(n * M + 1, dtype=np.uint64)
    np.cumsum(lens.reshape(-1), out=q_off[1:])
    waits = np.zeros(int(q_off[-1]), dtype=np.uint32)
    for m in range(M):
        lam = float(rate_per_us[m])
        keys = stream_key(seed, scen_ids, m, STREAM_SNAPSHOT)
        cum = _unit_gaps_cum(keys, depth_max) / lam  # newest task first
        for j in range(n):
            k = int(lens[j, m])
            if k:
                w = np.floor(cum[j, :k]).astype(np.uint32)
                waits[q_off[j * M + m]:q_off[j * M + m + 1]] = w[::-1]
    return q_off, waits


def harvest_snapshots(traces, n_dec, dec_cap, dec_t, dec_m, dec_B, max_snap=None):
    """Queue snapshots at the decision instants of a replay log (any
    scheduler's: the caller passes its per-scenario decision times, chosen
    models and batch sizes, log stride dec_cap).  Snapshot k of scenario s
    holds, per model m, the waits t_k - a of the requests of Q_m that arrived
    by t_k (a <= t_k, reading Q10) and were not yet dispatched (the dispatched
    ones are the first sum of B over earlier decisions on m).  Pure indexing,
    no scheduling arithmetic.  Returns (q_off u64 [n*M+1], waits u32, cfg_idx
    u16 [n]) in scenario-major, decision order."""
    M = traces.M
    q_lens, parts, ci = [], [], []
    taken = 0
    for s in range(traces.n_scen):
        k = int(n_dec[s])
        if max_snap is not None:
            k = min(k, max_snap - taken)
        if k <= 0:
            break
        t = dec_t[s * dec_cap:s * dec_cap + k].astype(np.int64)
        dm = dec_m[s * dec_cap:s * dec_cap + k].astype(np.int64)
        dB = dec_B[s * dec_cap:s * dec_cap + k].astype(np.int64)
        lens = np.zeros((k, M), np.int64)
        per_m = []
        for m in range(M):
            arr = traces.arrival[int(traces.arr_off[s * M + m]):int(traces.arr_off[s * M + m + 1])].astype(np.int64)
            tail = np.searchsorted(arr, t, side="right")
            served = np.where(dm == m, dB, 0)
            head = np.cumsum(served) - served  # dispatched before decision k
            ln = np.maximum(tail - head, 0)
            lens[:, m] = ln
            # flat gather: for each snapshot, arr[head:head+ln]
            tot = int(ln.sum())
            start = np.repeat(head - (np.cumsum(ln) - ln), ln)
            idx = np.arange(tot, dtype=np.int64) + start
            per_m.append((ln, t.repeat(ln) - arr[idx]))
        # interleave: snapshot-major, model-minor
        seg_len = lens.reshape(-1)
        out = np.empty(int(seg_len.sum()), np.uint32)
        dst_off = np.concatenate([[0], np.cumsum(seg_len)[:-1]]).reshape(k, M)
        for m in range(M):
            ln, w = per_m[m]
            dst = np.repeat(dst_off[:, m] - (np.cumsum(ln) - ln), ln) + np.arange(int(ln.sum()), dtype=np.int64)
            out[dst] = w
        q_lens.append(seg_len)
        parts.append(out)
        ci.append(np.full(k, int(traces.cfg_idx[s]), np.uint16))
        taken += k
    seg = np.concatenate(q_lens).astype(np.uint64)
    q_off = np.zeros(seg.size + 1, np.uint64)
    np.cumsum(seg, out=q_off[1:])
    return q_off, np.concatenate(parts), np.concatenate(ci)


# --------------------------------------------------------------------------- workloads


@dataclass
class Workload:
    name: str
    profile: Profile
    cfgs: list
    traces: Traces
    n_req: int
    desc: str = ""


def workload(name: str, scen_ids=None, n_req=None, seed=None) -> Workload:
    """North-star configs (BASELINE.json configs[0..4]) as concrete inputs.

    scen_ids selects a subset of the config's scenarios (global ids); n_req
    overrides the per-scenario request count (tests only; bench uses defaults).
    """
    if name == "cfg1":  # 1 scenario, 3x3x{1,2,4,8}, 1,000 requests, 50 ms, rho 1.0
        prof = synth_profile(3, 3, [1, 2, 4, 8])
        cfgs = [SchedCfg(tau=50000, b_max=8)]
        total = 1
        cfg_of = lambda s: 0
        rho_of = lambda s: 1.0
        group_of = lambda s: 0
        n_req_d, seed_d, kind = 1000, 7, "poisson"
    elif name == "cfg2":  # 4,096 scen, 4x4x16, 10k req, Poisson rho 0.60..1.20
        prof = synth_profile(4, 4, list(range(1, 17)))
        cfgs = [SchedCfg(tau=50000, b_max=16)]
        total = 4096
        cfg_of = lambda s: 0
        rho_of = lambda s: 0.60 + 0.05 * (s % 13)
        group_of = lambda s: s % 13
        n_req_d, seed_d, kind = 10000, 2, "poisson"
    elif name == "cfg3":  # 65,536 scen, 8x5x32, MMPP, tau 20..100 ms
        prof = synth_profile(8, 5, list(range(1, 33)))
        cfgs = [SchedCfg(tau=20000 + 10000 * k, b_max=32) for k in range(9)]
        total = 65536
        cfg_of = lambda s: s % 9
        rho_of = lambda s: 0.60 + 0.05 * ((s // 9) % 13)
        group_of = lambda s: (s % 9) * 13 + (s // 9) % 13
        n_req_d, seed_d, kind = 10000, 3, "mmpp"
    elif name == "cfg4":  # 1M scen sweep: 16 tau x 16 rho x 4096 seeds
        prof = synth_profile(4, 4, list(range(1, 17)))
        cfgs = [SchedCfg(tau=20000 + 5000 * k, b_max=16) for k in range(16)]
        total = 1 << 20
        cfg_of = lambda s: s % 16
        rho_of = lambda s: 0.60 + 0.06 * ((s // 16) % 16)
        group_of = lambda s: s % 256
        n_req_d, seed_d, kind = 10000, 4, "poisson"
    elif name == "cfg5a":  # 262,144 scen, 1M-request traces, rho_full 1.5
        prof = synth_profile(8, 5, list(range(1, 33)))
        cfgs = [SchedCfg(tau=50000, b_max=32)]
        total = 262144
        cfg_of = lambda s: 0
        rho_of = lambda s: 1.5
        group_of = lambda s: 0
        n_req_d, seed_d, kind = 1000000, 5, "poisson"
    elif name == "cfg5b":  # deep queues: rho_shallow 1.5
        prof = synth_profile(8, 5, list(range(1, 33)))
        cfgs = [SchedCfg(tau=50000, b_max=32)]
        total = 262144
        cfg_of = lambda s: 0
        rho_of = lambda s: 1.5
        group_of = lambda s: 0
        n_req_d, seed_d, kind = 50000, 6, "poisson_shallow"
    else:
        raise ValueError(f"unknown workload {name}")
    if scen_ids is None:
        scen_ids = np.arange(total, dtype=np.int64)
    scen_ids = np.asarray(scen_ids, dtype=np.int64)
    n_req = n_req_d if n_req is None else n_req
    seed = seed_d if seed is None else seed
    n = scen_ids.size
    M = prof.M
    lam = np.zeros((n, M))
    D = np.zeros(n)
    for j, s in enumerate(scen_ids):
        c = cfgs[cfg_of(int(s))]
        if kind == "poisson_shallow":
            lam[j] = rates_for_shallow_load(prof, c.b_max, rho_of(int(s)))
        else:
            lam[j] = rates_for_load(prof, c.b_max, rho_of(int(s)))
        D[j] = n_req / lam[j].sum()
    if kind == "mmpp":
        segs = mmpp_segments(seed, scen_ids, lam, D)
    else:
        segs = poisson_segments(seed, scen_ids, lam, D)
    tr = _assemble(M, segs, [cfg_of(int(s)) for s in scen_ids], [group_of(int(s)) for s in scen_ids],
                   scen_ids)
    return Workload(name=name, profile=prof, cfgs=cfgs, traces=tr, n_req=n_req,
                    desc=f"{name}: {kind}, {n} scenarios x ~{n_req} requests, M={M} E={prof.E} nb={prof.nb}")


def n_groups(name: str) -> int:
    return {"cfg1": 1, "cfg2": 13, "cfg3": 117, "cfg4": 256, "cfg5a": 1, "cfg5b": 1}[name]


def total_scenarios(name: str) -> int:
    return {"cfg1": 1, "cfg2": 4096, "cfg3": 65536, "cfg4": 1 << 20, "cfg5a": 262144,
            "cfg5b": 262144}[name]
