#!/usr/bin/env python
"""Benchmark: scheduling decisions/sec of the EdgeServing stability-score
engine (BASELINE.json metric) on BASELINE configs[1] (default workload cfg2:
4,096 scenarios x 4 DNNs x 4 exits x batch 1-16, 10k-request Poisson traces,
rho_full 0.60-1.20, tau = 50 ms).

One step = one pass of the whole hot path over the batch: K2 replay (a2-a8),
K3 per-scenario P95 (a9) and the per-group merge (a10; NCCL all_reduce across
ranks).  Inputs (164 MB of arrivals per rank) are resident in HBM and larger
than the 126 MB L2, so no extra flush is needed.  Multi-GPU: each rank replays
its own 4,096-scenario batch (weak scaling); only the group merge communicates.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scheduling decisions/sec (stability-score evals)"
UNIT = "decisions/s"


_OUT_FD = None


def emit(line):
    """The one JSON line on stdout.  Everything else the process (or NCCL's
    version banner) writes to fd 1 is redirected to stderr by main()."""
    os.write(_OUT_FD if _OUT_FD is not None else 1, (json.dumps(line) + "\n").encode())


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(PER_GPU))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: S scenarios per GPU; strong: S scenarios in total, split over the GPUs")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg2 line of the default cfg3 run")
    ap.add_argument("--scenarios", type=int, default=0, help="scenarios per GPU (default: PER_GPU[workload])")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-k1", action="store_true", help="skip the K1 snapshot-scoring measurement")
    ap.add_argument("--ncu", action="store_true", help="short run for ncu launch lists (no extras)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# per-GPU scenario counts (weak scaling) and descriptions of the BASELINE.json
# configs; cfg4 is the 1M-scenario sweep sharded over 8 GPUs, the two config-5
# readings run host-generated shards of 262,144 scenarios
PER_GPU = {"cfg1": 1, "cfg2": 4096, "cfg3": 65536, "cfg4": 131072, "cfg5a": 1024, "cfg5b": 16384}
DESC = {
    "cfg1": "cfg1 (BASELINE configs[0]): 1 scenario x 3 DNNs x 3 exits x batch {1,2,4,8}, 1,000-request Poisson trace, "
            "tau 50 ms",
    "cfg2": "cfg2 (BASELINE configs[1]): 4,096 scenarios/GPU x 4 DNNs x 4 exits x batch 1-16, 10k-request Poisson "
            "traces, rho 0.60-1.20, tau 50 ms",
    "cfg3": "cfg3 (BASELINE configs[2]): 65,536 scenarios/GPU x 8 DNNs x 5 exits x batch 1-32, 10k-request bursty "
            "MMPP traces, tau 20-100 ms x rho 0.60-1.20 (117 groups)",
    "cfg4": "cfg4 (BASELINE configs[3]): 1M-scenario SLO x rate sweep, 131,072 scenarios/GPU (1/8 shard) x 4 DNNs x "
            "4 exits x batch 1-16, 10k-request Poisson traces, 16 tau x 16 rho groups",
    "cfg5a": "cfg5-A (BASELINE configs[4], long-trace reading): 8 DNNs x 5 exits x batch 1-32, 1M-request Poisson "
             "traces at rho_full 1.5, 1,024-scenario shard/GPU",
    "cfg5b": "cfg5-B (BASELINE configs[4], deep-queue reading): 8 DNNs x 5 exits x batch 1-32, 50k-request traces at "
             "rho_shallow 1.5 (queues up to ~4k), 16,384-scenario shard/GPU",
}


def rank_workload(name, rank, S=None):
    """Weak scaling: rank r replays scenarios [r*S, (r+1)*S) of the config's
    scenario sequence (same generator, same shapes, distinct seeds)."""
    import inputs
    S = S or PER_GPU.get(name, inputs.total_scenarios(name))
    ids = np.arange(rank * S, (rank + 1) * S, dtype=np.int64)
    return inputs.workload(name, scen_ids=ids), S


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, bus_id):
        self.bus_id = bus_id
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.bus_id, f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.th.join(timeout=5)
        sm = []
        reasons = set()
        smax = None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
                for i, n in enumerate(names):
                    if r[4 + i].lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "samples": len(sm),
                "reasons": sorted(reasons)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6451.5), d.get("sm_max_mhz", 1965.0), "measured"
    return 6650.0, 1965.0, "fallback"


def ncu_traffic(kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(kernel)
    return None


def ncu_issue(kernel):
    """Issue-slot evidence of the last committed ncu --set full capture
    (smsp__issue_active, sm__inst_executed; profiles/ncu_traffic.json)."""
    return (ncu_traffic("_issue") or {}).get(kernel)


def alg_ops(stats_sum, requests, E):
    """Algorithmic integer operations of Algorithm 1 per the op model of
    DESIGN.md §6: 3 per Eq. 4 term (predicted-wait add, clip compare,
    accumulate), 7 per live task (w = t - a, urgency table lookup and
    product), 2 per examined (m, e) cell (Eq. 6 add + compare), 7 per
    candidate (Eq. 5 + score finalisation + Eq. 7 compare), 4 per request
    (admission compare, Eq. 1 latency, Eq. 2 compare, count), 2 per decision."""
    d, c, cells, live, terms = (stats_sum[k] for k in ("decisions", "candidates", "cells", "live", "terms"))
    return 3 * terms + 7 * live + 2 * cells + 7 * c + 4 * requests + 2 * d


def k1_batch(rank, n_gen=4096, tiles=64, depth=4096):
    """The K1 bench batch (host arrays): n_gen distinct seeded 5-C snapshots
    (inputs.snapshots_poisson_depth), repeated `tiles` times back to back in
    the flat CSR layout (snapshots are scored independently; the repetition
    only keeps host generation to seconds).  Shared by bench.py and the GPU
    test that samples it against the oracle."""
    import inputs
    rate = [depth / 120000.0] * 8
    q0, w0 = inputs.snapshots_poisson_depth(1000 + rank, np.arange(n_gen), 8, depth, rate)
    nw = np.uint64(w0.size)
    q_off = np.concatenate([q0[:-1] + np.uint64(t) * nw for t in range(tiles)] + [q0[-1:] + np.uint64(tiles - 1) * nw])
    return q_off, w0, tiles


def k1_time(es, h, dq, dw, dci, dev, stream, iters=10):
    """Mean device time of one es_score_candidates call (CUDA events on the
    launching stream, L2 flushed between launches) and the call's outputs."""
    import torch
    out = es.es_score_candidates(h, dq, dw, dci, stream=stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ms = []
    for i in range(iters + 2):
        flush.fill_(i & 0xFF)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        es.es_score_candidates(h, dq, dw, dci, out=out, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ms.append(a.elapsed_time(b))
    return statistics.mean(ms) / 1e3, out


def k1_line(es, h, M, q_off, w0, tiles, ci, x_c, dev, stream, desc, kernel, traffic_key, iters=10):
    """One K1 bench object: the distinct snapshots (q_off, w0, ci) repeated
    `tiles` times back to back; algorithmic bytes = per snapshot the M+1 queue
    offsets (8 B), the cfg index (2 B, when present) and the outputs (m, e, B,
    L, S, flags and M candidate scores: 17 + 8 M B), plus 4 B per LIVE wait
    (w < x_c of its cfg; the clipped prefix is counted from the index, never
    read -- P:309 clip, Q24)."""
    import torch
    n0 = (q_off.size - 1) // M
    nw = np.uint64(w0.size)
    q = np.concatenate([q_off[:-1] + np.uint64(t) * nw for t in range(tiles)] + [q_off[-1:] + np.uint64(tiles - 1) * nw])
    n_snap = n0 * tiles
    dq = torch.from_numpy(q).to(dev)
    dw = torch.from_numpy(w0).to(dev).repeat(tiles)
    dci = None if ci is None else torch.from_numpy(np.tile(ci, tiles)).to(dev)
    # live waits: per snapshot, waits below its cfg's x_c
    if ci is None:
        n_live = int((w0 < x_c[0]).sum()) * tiles
    else:
        snap_of_wait = np.repeat(np.arange(n0), np.diff(q_off[::M].astype(np.int64)))
        n_live = int((w0 < np.asarray(x_c, np.uint64)[ci[snap_of_wait]]).sum()) * tiles
    t_s, out = k1_time(es, h, dq, dw, dci, dev, stream, iters)
    alg = n_snap * (8 * (M + 1) + (2 if ci is not None else 0) + 17 + 8 * M) + 4 * n_live
    hbm, _, src = peaks()
    flags = out["flags"].cpu().numpy()
    return {"workload": desc + f" ({n_snap} snapshots, {w0.size * tiles} waits of which {n_live} live, "
                               f"{w0.nbytes * tiles / 1e6:.0f} MB; {n0} distinct x {tiles})",
            "snapshots_per_s": n_snap / t_s, "scored_candidates_per_s": float((out["cand"] != 0xFFFFFFFFFFFFFFFF)
                                                                             .sum().item()) / t_s,
            "ms_per_launch": t_s * 1e3, "feasible_frac": float((flags & 1).mean()),
            "roofline": {"bound": "hbm", "achieved": alg / t_s / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": alg / t_s / 1e9 / hbm, "traffic": ncu_traffic(traffic_key),
                         "kernel": kernel, "alg_bytes_per_launch": alg,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})", "l2": "flushed between launches"}}


def bench_k1(es, dev, stream, rank, depth=4096):
    """K1 (es_score_candidates) on 5-C-shaped snapshots: M=8, E=5, batch 1-32,
    per-model depth U[0, 4096], waits = t - Poisson arrivals in FIFO order.
    Rates are set so a full queue spans ~120 ms < x_c - max L: every task is in
    the live window and is read (the HBM-streaming regime).  262,144 snapshots
    (17.3 GB of waits: SURVEY 5-C's full size; k1_batch)."""
    import inputs
    prof = inputs.synth_profile(8, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
    q_off, w0, tiles = k1_batch(rank, depth=depth)
    h = es.es_load_profile(prof, cfgs, device=dev.index)
    x_c = [es.es_get_tables(h, 0)["x_c"]]
    n0 = (q_off.size - 1) // 8 // tiles
    return k1_line(es, h, 8, q_off[:n0 * 8 + 1], w0, tiles, None, x_c, dev, stream,
                   f"5-C shape: 8 DNNs x 5 exits x batch 1-32, depth U[0,{depth}] per model, all tasks live",
                   "k1 call: k1s_prep + k1s_stream_tma + k1s_clip + k1s_finish", "k1_call")


def bench_k1_clip(es, dev, stream, rank, depth=4096):
    """K1 on 5-C depth under 5-B's overload rates (rates_for_shallow_load,
    rho 1.5): queue heads wait past x_c - max L, so every snapshot takes the
    general per-candidate clip path and long clipped prefixes are
    counted, not read."""
    import inputs
    prof = inputs.synth_profile(8, 5, list(range(1, 33)))
    cfgs = [inputs.SchedCfg(tau=50000, b_max=32)]
    rate = inputs.rates_for_shallow_load(prof, 32, 1.5)
    q_off, w0 = inputs.snapshots_poisson_depth(2000 + rank, np.arange(4096), 8, depth, rate)
    h = es.es_load_profile(prof, cfgs, device=dev.index)
    x_c = [es.es_get_tables(h, 0)["x_c"]]
    return k1_line(es, h, 8, q_off, w0, 64, None, x_c, dev, stream,
                   f"5-C depth U[0,{depth}] at 5-B overload rates (rho_shallow 1.5): heads past x_c - max L, "
                   "the general clip path", "k1 call (clip path)", "k1_clip")


def k1_harvested_batch(es, engine, dev, stream, rank, n_scen=512):
    """The harvested cfg3 snapshots (host arrays) and a profile handle: n_scen
    cfg3 scenarios replayed by K2 with the decision log on, every decision's
    queue state rebuilt on the host (inputs.harvest_snapshots, pure indexing)."""
    import torch
    import inputs
    w = inputs.workload("cfg3", scen_ids=np.arange(rank * n_scen, (rank + 1) * n_scen))
    h = es.es_load_profile(w.profile, w.cfgs, device=dev.index)
    d = engine.upload_traces(w.traces, dev)
    cap = int(max(np.diff(w.traces.arr_off.astype(np.int64)[::w.profile.M])))  # <= one decision per request
    o = es.es_replay_traces(h, d["arr_off"], d["arrival"], d["cfg_idx"], d["group_id"], full=True, p95=False,
                            dec_cap=cap, stream=stream)
    torch.cuda.synchronize()
    n_dec = o["stats"][:, 0].cpu().numpy()
    q_off, w0, ci = inputs.harvest_snapshots(w.traces, n_dec, cap, o["dec_t"].cpu().numpy(),
                                             o["dec_m"].cpu().numpy(), o["dec_B"].cpu().numpy())
    del o, d
    x_c = [es.es_get_tables(h, k)["x_c"] for k in range(len(w.cfgs))]
    return h, q_off, w0, ci, x_c


def bench_k1_harvested(es, engine, dev, stream, rank, n_scen=512, tiles=8, batch=None):
    """K1 on queue snapshots harvested at the decision instants of cfg3
    replays ('harvested config-3 snapshots', k1_harvested_batch),
    nine SLO configs mixed by the snapshots' cfg index."""
    h, q_off, w0, ci, x_c = batch or k1_harvested_batch(es, engine, dev, stream, rank, n_scen)
    live_per = float(np.mean(np.diff(q_off[::8].astype(np.int64))))
    return k1_line(es, h, 8, q_off, w0, tiles, ci, x_c, dev, stream,
                   f"cfg3 harvested: every decision instant of {n_scen} cfg3 scenarios (8 DNNs x 5 exits x batch "
                   f"1-32, 9 SLOs), {live_per:.1f} queued tasks per snapshot on average",
                   "k1 call (thread per snapshot)", "k1_harvested")


def run_reference(args, rank, world):
    """--impl reference: the oracle (plain C, CPU) as it stands on the host cores."""
    if rank != 0:
        return
    import oracle
    import inputs
    S = args.scenarios or PER_GPU[args.workload]
    cores = os.cpu_count() or 1
    per = inputs.workload(args.workload, scen_ids=np.arange(1)).traces.arrival.size  # requests per scenario
    chunk = int(max(1, min(512, S, 5e6 // per)))
    nsteps = args.warmup + args.steps
    times = []
    dec = 0
    for k in range(nsteps):
        lo = (k * chunk) % S
        ids = np.arange(lo, lo + chunk)
        sub = inputs.workload(args.workload, scen_ids=ids)
        t0 = time.perf_counter()
        o = oracle.replay_batch(sub.profile, sub.cfgs, sub.traces, full=False, nthreads=cores)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
            dec += int(o["stats"][:, 0].sum())
    tot = sum(times)
    v = dec / tot
    sample = f"{chunk} scenarios of {args.workload} per step (cycling through the {S}-scenario batch), full traces"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": DESC[args.workload], "scenarios_per_step": chunk},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def init_dist(dev, world):
    """One process per GPU; the NCCL process group is created at every N
    (N = 1 included), so the group merge's all_reduce always runs through NCCL."""
    import socket
    import torch.distributed as dist
    if "MASTER_ADDR" not in os.environ:  # plain `python bench.py` (N = 1, no torchrun)
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=dev)
    return dist.group.WORLD


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def main():
    global _OUT_FD
    args = parse()
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)  # stray prints (NCCL's banner included) go to stderr
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    import paper_2605_05527_b200 as es
    from paper_2605_05527_b200 import engine

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = init_dist(dev, world)
    import inputs

    # weak scaling (default): each rank replays its own S-scenario batch of the
    # config's sequence; strong: a fixed S-scenario batch split over the ranks
    S_cfg = args.scenarios or PER_GPU[args.workload]
    if args.scaling == "strong":
        ids = engine.shard_ids(S_cfg, rank, world)
        w = inputs.workload(args.workload, scen_ids=ids)
        S = int(ids.size)
    else:
        w, S = rank_workload(args.workload, rank, args.scenarios)
    G = inputs.n_groups(args.workload)
    h = es.es_load_profile(w.profile, w.cfgs, device=local)
    dtr = engine.upload_traces(w.traces, dev)
    total = int(w.traces.arrival.size)
    out = es.alloc_replay_out(h, S, total, dev, full=False, p95=True)
    stream = torch.cuda.current_stream()
    ev = {"k2": [], "k3": [], "merge": []}

    def step(record):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if record else None
        if record:
            e[0].record(stream)
        es.es_replay_traces(h, dtr["arr_off"], dtr["arrival"], dtr["cfg_idx"], dtr["group_id"], out=out,
                            full=False, p95=False, stream=stream)
        if record:
            e[1].record(stream)
        # K3 (per-scenario P95) fused with the level-0 group histogram, then the
        # NCCL all_reduce'd radix levels of the exact group P95 (engine.group_merge)
        counts, p95g = engine.group_merge(h, dtr, out, G, group=pg, stream=stream, with_p95=True,
                                          events=e[2:] if record else None)
        if record:
            ev["k2"].append((e[0], e[1]))
            ev["k3"].append((e[1], e[2]))
            ev["merge"].append((e[2], e[3]))
        return counts, p95g

    for _ in range(max(args.warmup, 1)):
        counts, p95g = step(False)
    torch.cuda.synchronize()
    st = out["stats"].cpu().numpy()
    assert int(st[:, 7].max()) == 0, "a scenario reported an error status"
    cols = es.STAT_COLS
    ssum = {c: int(st[:, i].sum()) for i, c in enumerate(cols)}
    decisions_rank = ssum["decisions"]
    cand_rank = ssum["candidates"]

    # ---------------- timed region (device events, max over ranks)
    bus = None
    try:
        p = torch.cuda.get_device_properties(dev)
        bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
    except Exception:
        pass
    sampler = ClockSampler(bus) if (bus and not args.ncu) else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    l0 = h.launches
    dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(True)
    t1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop() if sampler else None
    launches = h.launches - l0 + 4 * args.steps  # + the four group-select kernels per step
    ms = t0.elapsed_time(t1)
    kms = {k: statistics.mean(a.elapsed_time(b) for a, b in v) for k, v in ev.items()}
    tt = torch.tensor([ms, float(decisions_rank), float(cand_rank)], dtype=torch.float64, device=dev)
    mx = tt[:1].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tt[1:].clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    ms_max, dec_all, cand_all = float(mx[0]), float(sm[0]), float(sm[1])
    value = dec_all * args.steps / (ms_max / 1e3)

    # ---------------- roofline of the dominant kernel (K2) -- issue/ALU bound
    hbm, sm_max, src = peaks()
    k2_avg_s = kms["k2"] / 1e3
    ops = alg_ops(ssum, total, w.profile.E)
    peak_ops = 148 * 128 * sm_max * 1e6  # 148 SMs x 4 schedulers x 32 lanes x clock (SURVEY 8(d) issue peak)
    achieved = ops / k2_avg_s
    alg_bytes = 4 * total + 4 * total + 8 * es.ES_NSTAT * S + 8 * (S * w.profile.M + 1)
    roof = {"bound": "alu", "achieved": achieved / 1e9, "peak": peak_ops / 1e9, "unit": "Gop/s",
            "frac": achieved / peak_ops,
            "traffic": ncu_traffic("k2_replay_" + args.workload) or (ncu_traffic("k2_replay") if args.workload == "cfg3"
                                                                      else None),
            "kernel": "k2_replay", "k2_ms": kms["k2"], "k2_share_of_step": kms["k2"] / (ms / args.steps),
            "peak_source": f"148 SM x 4 SMSP x 32 lanes x {sm_max:.0f} MHz ({src} sm_max): SURVEY 8(d)'s issue "
                           "peak in thread-instruction units",
            "alg_ops_per_launch": ops,
            "alg_ops_model": "DESIGN.md 6: 3 per Eq. 4 term + 7 per live task + 2 per examined (m,e) cell + 7 per "
                             "candidate + 4 per request + 2 per decision, counted exactly by the kernel",
            "hbm_view": {"alg_bytes_per_launch": alg_bytes, "achieved_gbs": alg_bytes / k2_avg_s / 1e9,
                         "peak_gbs": hbm, "frac": alg_bytes / k2_avg_s / 1e9 / hbm}}
    iss = ncu_issue("k2_replay") if args.workload == "cfg3" else None
    if iss and iss.get("warp_inst"):  # issue-slot evidence of the committed capture of this workload
        roof["issue_view"] = {"issue_active_pct": iss["issue_active_pct"], "warp_inst_per_launch": iss["warp_inst"],
                              "warp_inst_per_decision": iss["warp_inst"] / float(ssum["decisions"]),
                              "source": "profiles/ncu_traffic.json (_issue; ncu --set full of bench.py, "
                                        "profiles/r02_ncu_k2.txt)"}
    k3_bytes = 4 * total + 8 * es.ES_NSTAT * S  # K3 reads every latency once (+ the per-scenario counters)
    kernels = {"k2_ms": kms["k2"], "k3_ms": kms["k3"], "merge_ms": kms["merge"],
               "k3_gbs": k3_bytes / (kms["k3"] / 1e3) / 1e9,
               "merge_note": "group levels 1-3 (es_group_hist + NCCL all_reduce + es_group_p95_select)"}

    # chain view: K2 is bound by its longest dependent chain of decisions; the
    # longest scenario replayed alone on the GPU is that chain's latency floor
    if not args.ncu:
        s_max = int(np.argmax(st[:, 0]))
        w1 = inputs.workload(args.workload, scen_ids=np.array([int(w.traces.scen_ids[s_max])], np.int64))
        d1 = engine.upload_traces(w1.traces, dev)
        o1 = es.alloc_replay_out(h, 1, int(w1.traces.arrival.size), dev, full=False, p95=False)
        t1 = []
        for i in range(4):
            a1, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a1.record(stream)
            es.es_replay_traces(h, d1["arr_off"], d1["arrival"], d1["cfg_idx"], d1["group_id"], out=o1, full=False,
                                p95=False, stream=stream)
            b1.record(stream)
            torch.cuda.synchronize()
            if i:
                t1.append(a1.elapsed_time(b1))
        alone = statistics.median(t1)
        roof["chain_view"] = {"longest_chain_decisions": int(st[s_max, 0]), "alone_ms": alone,
                              "k2_ms": kms["k2"], "frac": alone / kms["k2"],
                              "cycles_per_decision_alone": alone * 1e-3 * sm_max * 1e6 / max(1, int(st[s_max, 0])),
                              "note": "longest scenario replayed alone = the batch's latency floor; frac = floor / K2"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": DESC[args.workload], "scenarios_per_gpu": S, "requests_per_gpu": total, "groups": G,
                       "l2": f"inputs larger than L2 ({4 * total / 1e6:.0f} MB arrivals/GPU > 126 MB)"
                             if 4 * total > 126e6 else f"inputs fit L2 ({4 * total / 1e6:.1f} MB arrivals/GPU)",
                       "parallelism": f"scenario-sharded x{world} ({args.scaling} scaling), NCCL all_reduce of "
                                      "group counters and histograms"},
            "scored_candidates_per_s": cand_all * args.steps / (ms_max / 1e3),
            "decisions_per_step": dec_all, "gpu_launches": launches, "kernels": kernels, "roofline": roof}
    if clocks:
        line["clocks"] = clocks

    # ---------------- e2e: the same step through the public host-memory API
    # (engine.replay_group_stats_host: pinned H2D of every step's traces,
    # K2 + K3 + the NCCL group merge, D2H of counters and P95s)
    if not args.no_e2e and not args.ncu:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        tr = w.traces
        hin = {"arr_off": pin(tr.arr_off.view(np.int64)).view(torch.uint64),
               "arrival": pin(tr.arrival.view(np.int32)).view(torch.uint32),
               "cfg_idx": pin(tr.cfg_idx.view(np.int16)).view(torch.uint16),
               "group_id": pin(tr.group_id.view(np.int32)).view(torch.uint32)}
        mk = lambda: {"stats": torch.empty((S, es.ES_NSTAT), dtype=torch.uint64).pin_memory(),
                      "p95": torch.empty(S, dtype=torch.uint32).pin_memory(),
                      "counts": torch.empty((G, es.ES_NGSTAT), dtype=torch.uint64).pin_memory(),
                      "gp95": torch.empty(G, dtype=torch.uint64).pin_memory()}
        n_e2e = max(3, min(args.steps, 20))
        houts = [mk(), mk()]
        engine.replay_group_stats_host(h, [(hin, houts[0])], G, group=pg, stream=stream)  # warm
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        a = time.perf_counter()
        e0.record(stream)
        engine.replay_group_stats_host(h, [(hin, houts[k & 1]) for k in range(n_e2e)], G, group=pg, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        wall_ms = (time.perf_counter() - a) * 1e3
        et = torch.tensor([max(e_ms, wall_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_v = dec_all * n_e2e / (float(et[0]) / 1e3)
        h2d = sum(int(x.numel() * x.element_size()) for x in hin.values())
        d2h = sum(int(x.numel() * x.element_size()) for x in houts[0].values())
        assert np.array_equal(houts[0]["stats"].numpy(), st)
        assert np.array_equal(houts[0]["counts"].numpy(), counts.cpu().numpy())
        assert np.array_equal(houts[0]["gp95"].numpy(), p95g.cpu().numpy())
        line["e2e"] = {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "steps": n_e2e,
                       "call": "engine.replay_group_stats_host (pinned host traces in, per-scenario counters + P95 "
                               "and group counters + P95 out, every step; K2 + K3 + NCCL group merge; step k+1's "
                               "H2D overlaps step k)"}

    # ---------------- K1: independent snapshot scoring, the HBM-streaming form
    if not args.no_k1 and not args.ncu:
        line["k1"] = bench_k1(es, dev, stream, rank)
        line["k1_clip"] = bench_k1_clip(es, dev, stream, rank)
        line["k1_harvested"] = bench_k1_harvested(es, engine, dev, stream, rank)

    # ---------------- the other configs' headline lines (K2 + K3 + merge per step)
    if args.workload == "cfg3" and not args.no_extra and not args.ncu:
        line["cfg2"] = bench_extra("cfg2", es, engine, dev, stream, pg, rank)

    # ---------------- CPU baseline: the oracle on the host cores (rank 0, N=1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.ncu:
        line["cpu_baseline"] = cpu_baseline(args, w, S, total, st, out)
    if rank == 0:
        emit(line)
    dist.destroy_process_group()


def bench_extra(name, es, engine, dev, stream, pg, rank, steps=20):
    """Another config's step (K2 + K3 + NCCL group merge), device-timed."""
    import torch
    import inputs
    w, S = rank_workload(name, rank)
    G = inputs.n_groups(name)
    h = es.es_load_profile(w.profile, w.cfgs, device=dev.index)
    d = engine.upload_traces(w.traces, dev)
    o = es.alloc_replay_out(h, S, int(w.traces.arrival.size), dev, full=False, p95=True)
    for _ in range(3):
        engine.replay_group_stats(h, d, G, group=pg, stream=stream, out=o)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        engine.replay_group_stats(h, d, G, group=pg, stream=stream, out=o)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    dec = float(o["stats"][:, 0].sum().item())
    return {"workload": DESC[name], "value": dec / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "decisions_per_step": dec}


def cpu_baseline(args, w, S, total, st, out):
    """The oracle as it stands on the host cores: all cores on a bounded sample
    (bit-exact check against the GPU on it) and one core on a smaller one."""
    import inputs
    import oracle
    cores = os.cpu_count() or 1
    per = total / S
    k = S if total <= 50e6 else max(1, int(50e6 // per))  # <= ~50M requests
    ws = w if k == S else inputs.workload(args.workload, scen_ids=w.traces.scen_ids[:k])
    reps = 0
    t = time.perf_counter()
    while True:  # >= ~1 s wall (~16 s of CPU work on 16 cores)
        o = oracle.replay_batch(ws.profile, ws.cfgs, ws.traces, full=False, nthreads=cores)
        reps += 1
        if time.perf_counter() - t > 1.0:
            break
    dt = (time.perf_counter() - t) / reps
    assert np.array_equal(o["stats"], st[:k]), "oracle and GPU disagree on the bench batch"
    assert np.array_equal(o["p95"], out["p95"].cpu().numpy()[:k])
    k1 = max(1, min(k, int(2e6 // per)))  # single thread: ~2M requests
    w1 = inputs.workload(args.workload, scen_ids=w.traces.scen_ids[:k1])
    t = time.perf_counter()
    o1 = oracle.replay_batch(w1.profile, w1.cfgs, w1.traces, full=False, nthreads=1)
    dt1 = time.perf_counter() - t
    what = f"the full {S}-scenario bench batch" if k == S else f"the first {k} of the {S} bench scenarios"
    return {"value": int(o["stats"][:, 0].sum()) / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{what} (rank 0), {reps} replay(s), {dt:.2f} s wall each on {cores} threads",
            "parity": f"bit-exact on all per-scenario counters and P95 of those {k} scenarios",
            "single_thread": {"value": int(o1["stats"][:, 0].sum()) / dt1, "unit": UNIT, "cores": 1,
                              "sample": f"the first {k1} scenarios, {dt1:.2f} s on 1 thread"}}


if __name__ == "__main__":
    main()
