"""K2 alone on the bench's cfg3 batch (65,536 scenarios, inputs generated once)
for several prebuilt library variants (paths as arguments; 'default' = the
in-tree library): mean K2 ms over a few calls and decisions/s; every variant's
per-scenario counters must equal the first one's (bit-exact)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import inputs
import paper_2605_05527_b200 as es
from paper_2605_05527_b200 import engine

n = int(os.environ.get("NSCEN", "65536"))
wl = os.environ.get("WL", "cfg3")
t0 = time.time()
w = inputs.workload(wl, scen_ids=np.arange(n))
dtr = engine.upload_traces(w.traces, "cuda")
print(f"{wl} {n} scenarios generated in {time.time() - t0:.0f} s", flush=True)
ref = None
for spec in sys.argv[1:] or ["default"]:
    v, _, envs = spec.partition("+")
    for kv in filter(None, envs.split(",")):
        os.environ[kv.split("=")[0]] = kv.split("=")[1]
    es._lib = None
    es.LIB_PATH = os.path.join(ROOT, "paper_2605_05527_b200", "libedgeserve.so") if v == "default" else os.path.abspath(v)
    h = es.es_load_profile(w.profile, w.cfgs)
    out = es.es_replay_traces(h, dtr["arr_off"], dtr["arrival"], dtr["cfg_idx"], dtr["group_id"], full=False, p95=False)
    ms = []
    for i in range(4):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        es.es_replay_traces(h, dtr["arr_off"], dtr["arrival"], dtr["cfg_idx"], dtr["group_id"], out=out, full=False,
                            p95=False)
        b_.record()
        torch.cuda.synchronize()
        ms.append(a_.elapsed_time(b_))
    st = out["stats"].cpu().numpy()
    same = "ref" if ref is None else ("bit-exact" if np.array_equal(st, ref) else "DIFFERENT")
    if ref is None:
        ref = st
    dec = float(st[:, 0].sum())
    for kv in filter(None, envs.split(",")):
        os.environ.pop(kv.split("=")[0])
    print(f"{os.path.basename(spec):24s} K2 {np.mean(ms[1:]):8.3f} ms  {dec / np.mean(ms[1:]) * 1e3:.3e} decisions/s  {same}",
          flush=True)
