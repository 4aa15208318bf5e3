"""The multi-GPU path executed on the B200 through NCCL (one process per GPU,
launched by torchrun; world size 1 here -- gpurun exposes one GPU): the group
merge's all_reduce over a real NCCL communicator, compared bitwise with the
oracle, and the bench under torchrun (NCCL process group, barrier and
max-over-ranks timing) printing a valid line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, timeout):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port())] + args
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_nccl_group_merge_matches_oracle():
    r = _torchrun([os.path.join(ROOT, "tests", "dist", "nccl_merge.py")], 600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "NCCL_MERGE_OK world=1 backend=nccl" in r.stdout


def test_bench_under_torchrun_nccl():
    r = _torchrun([os.path.join(ROOT, "bench.py"), "--gpus", "1", "--workload", "cfg2", "--steps", "3", "--warmup",
                   "3", "--no-k1", "--no-cpu-baseline", "--no-e2e"], 900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    assert "NCCL" in line["config"]["parallelism"]
