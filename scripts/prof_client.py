"""Device time of the client-side calls of one end-to-end step (shard.run_sharded: encode, encrypt,
decrypt, decode) next to the server-side evaluation, from CUDA events around every engine call.

    python scripts/prof_client.py [--batch 64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_03060_b200 import _lib, planner, shard  # noqa: E402
from paper_2402_03060_b200.he_backend import GpuBackend  # noqa: E402
from paper_2402_03060_b200.params import HEParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    args = ap.parse_args()
    params = HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=2)
    m = planner.lenet1(0)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    imgs = np.random.default_rng(0).uniform(0, 1, size=(args.batch * plan.capacity, 1, 28, 28))
    for _ in range(2):
        shard.run_sharded(m, imgs, params, be, plan=plan)
    torch.cuda.synchronize()
    _lib.PROFILE = []
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    shard.run_sharded(m, imgs, params, be, plan=plan)
    s1.record()
    torch.cuda.synchronize()
    total = s0.elapsed_time(s1)
    print(f"e2e step {total:.2f} ms (device events around run_sharded)")
    for name, calls, ms in _lib.profile_summary(_lib.PROFILE):
        print(f"  {name:28s} {calls:5d} calls {ms:9.3f} ms")
    _lib.PROFILE = None


if __name__ == "__main__":
    main()
