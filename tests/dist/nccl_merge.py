"""Run under torchrun (one process per GPU, NCCL): each rank replays its shard
of a cfg2 subset, engine.group_merge all_reduces the group counters and radix
histograms over NCCL (group=WORLD), and rank 0 compares the merged counters
and group P95s bitwise with the oracle on the whole subset."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_2605_05527_b200 as es  # noqa: E402
from paper_2605_05527_b200 import engine  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n = 78
    ids = engine.shard_ids(n, rank, world)
    w = inputs.workload("cfg2", scen_ids=ids, n_req=1500)
    h = es.es_load_profile(w.profile, w.cfgs, device=local)
    d = engine.upload_traces(w.traces, dev)
    out, counts, p95 = engine.replay_group_stats(h, d, 13, group=dist.group.WORLD)
    torch.cuda.synchronize()
    assert dist.get_backend() == "nccl"
    if rank == 0:
        wa = inputs.workload("cfg2", scen_ids=np.arange(n), n_req=1500)
        o = oracle.replay_batch(wa.profile, wa.cfgs, wa.traces, nthreads=8)
        oc, op = oracle.group_stats(wa.traces, o, wa.cfgs, 13)
        assert np.array_equal(counts.cpu().numpy(), oc), "merged counters differ"
        assert np.array_equal(p95.cpu().numpy().astype(np.uint32), op), "group P95 differs"
        print(f"NCCL_MERGE_OK world={world} backend={dist.get_backend()}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
