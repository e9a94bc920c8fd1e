"""Build a compile-time variant of the engine next to the default one, for A/B timing.

    python scripts/build_variant.py NAME [-DKNOB=VALUE ...] [--only file.cu ...]

compiles csrc/*.cu with the extra defines into paper_2402_03060_b200/_build/var_NAME/ and links
libunihenn_b200.so there; run either build with UH_LIB_PATH=<that .so> (see _lib.py).  Sources not
listed under --only reuse the default build's objects (the knobs are file-local macros).
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_03060_b200 import build as B  # noqa: E402


def main():
    name = sys.argv[1]
    args = sys.argv[2:]
    only = []
    if "--only" in args:
        i = args.index("--only")
        only = args[i + 1:]
        args = args[:i]
    defs = [a for a in args if a.startswith("-D")]
    B.build()
    out = os.path.join(B.OUT_DIR, "var_" + name)
    os.makedirs(out, exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    srcs = B.sources()
    mine = [s for s in srcs if not only or os.path.basename(s) in only]

    def obj(s):
        return os.path.join(out if s in mine else B.OUT_DIR, os.path.basename(s)[:-3] + ".o")

    def cc(s):
        subprocess.run([nvcc, *B.ARCH, *B.NVCC_FLAGS, *defs, "-c", "-o", obj(s), s], check=True)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(cc, mine))
    lib = os.path.join(out, "libunihenn_b200.so")
    subprocess.run([nvcc, *B.ARCH, "-shared", "-ccbin", "/usr/bin/g++", "-o", lib, *[obj(s) for s in srcs]], check=True)
    print(lib)


if __name__ == "__main__":
    main()
