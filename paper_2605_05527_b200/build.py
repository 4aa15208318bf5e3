"""Build libedgeserve.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libedgeserve.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, ptxas_v=False, lib=None, defines=()):
    """Compile every csrc/*.cu and link the shared library (`lib`, default the
    in-tree libedgeserve.so).  `defines` are extra -D flags (tuning variants)."""
    lib = lib or LIB
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "edgeserve.h")]
    if not force and not _stale(lib, deps):
        return lib
    objdir = os.path.join(HERE, "build" if lib == LIB else "build_" + os.path.basename(lib)[:-3])
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *["-D" + d for d in defines], "-c", src, "-o", obj]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(obj)
    # exported symbols: the es_* C ABI (api.cu marks them default visibility)
    cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fPIC"]
    subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [--lib PATH -DNAME=V ...]
    args = sys.argv[1:]
    lib = args[args.index("--lib") + 1] if "--lib" in args else None
    defs = [x[2:] for x in args if x.startswith("-D")]
    build(force="--force" in args, verbose=True, ptxas_v="-v" in args, lib=lib, defines=defs)
