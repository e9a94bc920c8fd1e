"""Wall-clock split of driver.infer_batch (the bench's e2e path) into its stages.

    python scripts/prof_e2e.py [--batch 64]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_03060_b200 import driver, planner  # noqa: E402
from paper_2402_03060_b200.driver import CostModel, _extract, _input_layout, _run_layers  # noqa: E402
from paper_2402_03060_b200.he_backend import GpuBackend  # noqa: E402
from paper_2402_03060_b200.params import HEParams  # noqa: E402
from paper_2402_03060_b200.schedule import CipherState  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    args = ap.parse_args()
    params = HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=2)
    m = planner.lenet1(0)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    rng = np.random.default_rng(0)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28))) for _ in range(args.batch)]
    planes = driver.pack_groups(m, groups, plan)
    for _ in range(2):
        driver.infer_batch(m, planes, params, plan, be, fused=True)
    torch.cuda.synchronize()
    t = {}

    def mark(name, t0):
        torch.cuda.synchronize()
        t[name] = t.get(name, 0.0) + time.perf_counter() - t0
        return time.perf_counter()

    reps = 3
    for _ in range(reps):
        t0 = time.perf_counter()
        planner.validate(m, params)
        t0 = mark("validate", t0)
        cts = [be.encrypt(be.encode_batch(planes[ch])) for ch in range(m.channels)]
        t0 = mark("encode+encrypt", t0)
        state, rows, total = _run_layers(m, CipherState(cts, _input_layout(m, plan)), be, CostModel(),
                                         params.poly_degree, True)
        t0 = mark("layers", t0)
        dec = [np.atleast_2d(be.decrypt(ct)) for ct in state.cts]
        t0 = mark("decrypt+D2H", t0)
        for b in range(dec[0].shape[0]):
            _extract([d[b] for d in dec], state.layout, plan.offsets[:plan.capacity])
        mark("extract", t0)
    for k, v in t.items():
        print(f"{k:16s} {1e3 * v / reps:9.3f} ms")


if __name__ == "__main__":
    main()
