"""Host-side enqueue time of one fused LeNet-1 step vs its device time (is the eager loop launch-bound?).

    python scripts/host_overhead.py [--batch 64]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_03060_b200 import driver, planner  # noqa: E402
from paper_2402_03060_b200.he_backend import GpuBackend  # noqa: E402
from paper_2402_03060_b200.params import HEParams  # noqa: E402
from paper_2402_03060_b200.schedule import CipherState  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    args = ap.parse_args()
    p = HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=2)
    m = planner.lenet1(0)
    plan = planner.footprint(m, p)
    be = GpuBackend(p)
    planes = driver.pack_groups(m, [list(np.random.default_rng(b).uniform(0, 1, size=(20, 1, 28, 28)))
                                    for b in range(args.batch)], plan)
    ct = [be.encrypt(be.encode_batch(planes[0]))]
    lay = driver._input_layout(m, plan)

    def step():
        return driver._run_layers(m, CipherState(ct, lay), be, driver.CostModel(), p.poly_degree, True)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    for k in range(5):
        t0 = time.perf_counter()
        step()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"step {k}: host enqueue {1e3 * (t1 - t0):7.1f} ms, until done {1e3 * (t2 - t0):7.1f} ms")
    import cProfile
    import pstats

    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    step()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
