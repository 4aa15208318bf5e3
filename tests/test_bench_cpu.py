"""bench.py's host-side pieces on CPU: the reference arm (the oracle timed on
the host cores, the base contract's --impl reference line) and the K1 batch
layout (tiled CSR consistent with the waits it indexes)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--workload", "cfg1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "decisions/s" and line["value"] > 0
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_k1_batch_layout():
    import bench
    q_off, w0, tiles = bench.k1_batch(0, n_gen=64, tiles=3, depth=64)
    M = 8
    assert q_off.size == 64 * tiles * M + 1
    assert int(q_off[0]) == 0 and int(q_off[-1]) == w0.size * tiles
    assert np.all(np.diff(q_off.astype(np.int64)) >= 0)
    # tile t of snapshot s indexes the same waits as snapshot s of tile 0
    lens = np.diff(q_off.astype(np.int64)).reshape(tiles, 64 * M)
    assert np.all(lens == lens[0])
