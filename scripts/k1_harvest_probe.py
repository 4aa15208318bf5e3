"""K1 on the harvested cfg3 batch (bench.bench_k1_harvested) under launch
variants given as ENV=VALUE,ENV=VALUE ... arguments (one bench object each)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_05527_b200 as es  # noqa: E402
from paper_2605_05527_b200 import engine  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
batch = bench.k1_harvested_batch(es, engine, dev, stream, 0, int(os.environ.get("NSCEN", "512")))
for v in sys.argv[1:] or [""]:
    for kv in filter(None, v.split(",")):
        k, x = kv.split("=")
        os.environ[k] = x
    o = bench.bench_k1_harvested(es, engine, dev, stream, 0, batch=batch)
    print(json.dumps({"variant": v, "ms": o["ms_per_launch"], "frac": o["roofline"]["frac"],
                      "snap_per_s": o["snapshots_per_s"]}), flush=True)
    for kv in filter(None, v.split(",")):
        os.environ.pop(kv.split("=")[0])
