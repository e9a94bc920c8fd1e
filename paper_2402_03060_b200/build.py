"""In-tree build of the sm_100a engine (and, for tests, the CPU oracle).

``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` over
``csrc/*.cu`` into ``_build/libunihenn_b200.so`` (git-ignored, travels to the
GPU box with the repo snapshot).  nvcc cross-compiles without a GPU.  Each
translation unit is compiled to its own object in parallel (a source is
recompiled when it, or any header, is newer than its object), then linked.
"""

from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libunihenn_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "unihenn_b200.h")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
              "-ccbin", "/usr/bin/g++"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]


def _obj(src: str) -> str:
    return os.path.join(OUT_DIR, os.path.basename(src)[:-3] + ".o")


def _newest(paths) -> float:
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _stale_objs(force: bool):
    hdr = _newest(_headers())
    out = []
    for s in sources():
        o = _obj(s)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr):
            out.append(s)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    todo = _stale_objs(force)

    def cc(src):
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-c", "-o", _obj(src), src]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    if todo:
        with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            list(ex.map(cc, todo))
    objs = [_obj(s) for s in sources()]
    # drop objects of deleted sources so they are never linked
    for o in glob.glob(os.path.join(OUT_DIR, "*.o")):
        if o not in objs:
            os.unlink(o)
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        cmd = [nvcc, *ARCH, "-shared", "-ccbin", "/usr/bin/g++", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose=True))
