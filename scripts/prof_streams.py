"""Device throughput of the LeNet-1 step with the batch split over S CUDA streams.

    python scripts/prof_streams.py [--batch 64] [--streams 1 2 4]

Each stream runs the whole fused network on its contiguous slice of the batch;
the MAC kernels (IMAD pipe) of one slice can then share SMs with the NTT
kernels (FP64 pipe) of another.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_03060_b200 import driver, planner  # noqa: E402
from paper_2402_03060_b200.he_backend import CipherVector, GpuBackend  # noqa: E402
from paper_2402_03060_b200.params import HEParams  # noqa: E402
from paper_2402_03060_b200.schedule import CipherState  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--streams", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    params = HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=2)
    m = planner.lenet1(0)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    rng = np.random.default_rng(0)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28))) for _ in range(args.batch)]
    planes = driver.pack_groups(m, groups, plan)
    ct = be.encrypt(be.encode_batch(planes[0]))
    layout = driver._input_layout(m, plan)
    main_stream = torch.cuda.current_stream()

    def run(S):
        B = ct.batch
        cuts = [B * k // S for k in range(S + 1)]
        streams = [torch.cuda.Stream() for _ in range(S)] if S > 1 else [main_stream]
        outs = []
        for k, st in enumerate(streams):
            st.wait_stream(main_stream)
            with torch.cuda.stream(st):
                sub = CipherVector(ct.data[cuts[k]:cuts[k + 1]], ct.level, ct.scale, be)
                state, _, _ = driver._run_layers(m, CipherState([sub], layout), be, driver.CostModel(),
                                                 params.poly_degree, True)
                outs.append(state.cts[0])
        for st in streams:
            main_stream.wait_stream(st)
        return outs

    for S in args.streams:
        for _ in range(2):
            run(S)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main_stream)
        for _ in range(args.steps):
            outs = run(S)
        e1.record(main_stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        d = np.concatenate([np.atleast_2d(be.decrypt(o)) for o in outs])
        ref = np.atleast_2d(be.decrypt(run(1)[0]))
        print(f"streams {S}: {ms:.2f} ms/step -> {args.batch * plan.capacity / (ms * 1e-3):.0f} images/s "
              f"(max |diff| vs 1 stream {np.max(np.abs(d - ref)):.2e})", flush=True)


if __name__ == "__main__":
    main()
