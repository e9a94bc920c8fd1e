"""Per-C-ABI-call and per-layer device time of one LeNet-1 step (B ciphertexts).

    python scripts/prof_step.py [--batch 16] [--oplevel]

Records CUDA events around every engine call (paper_2402_03060_b200._lib.PROFILE)
and around every layer, after warm-up; prints a table sorted by device time.
"""

import argparse
import os
import signal
import sys
import time

signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet when piped into head

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_03060_b200 import _lib, driver, fused, planner, schedule  # noqa: E402
from paper_2402_03060_b200.he_backend import GpuBackend  # noqa: E402
from paper_2402_03060_b200.params import HEParams  # noqa: E402
from paper_2402_03060_b200.schedule import CipherState  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--oplevel", action="store_true")
    ap.add_argument("--logn", type=int, default=15)
    ap.add_argument("--trace", action="store_true", help="print every engine call in order, per layer")
    ap.add_argument("--model", default="lenet1", help="planner builder: lenet1, cifar_net, config1_net, lr_model, svm_model")
    ap.add_argument("--depth", type=int, default=9)
    args = ap.parse_args()
    params = HEParams(poly_degree=1 << args.logn, depth=args.depth, scale_bits=40, seed=2)
    m = getattr(planner, args.model)(0)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    rng = np.random.default_rng(0)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, m.channels, m.height, m.width))) for _ in range(args.batch)]
    planes = driver.pack_groups(m, groups, plan)
    cts = [be.encrypt(be.encode_batch(planes[ch])) for ch in range(m.channels)]
    apply = schedule.apply_layer if args.oplevel else fused.apply_layer_fused
    need = sum(r.mults for r in planner.trace_layout(m))

    marks = []

    def step(layer_events=None):
        st = CipherState(cts, driver._input_layout(m, plan))
        st = schedule.drop_level(be, st, need)
        for layer in m.layers:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            if _lib.PROFILE is not None:
                marks.append((type(layer).__name__, len(_lib.PROFILE)))
            st = apply(be, st, layer)
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            if layer_events is not None:
                layer_events.append((type(layer).__name__, e0, e1))
        return st

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    _lib.PROFILE = []
    lev = []
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.profiler.start()  # `ncu --profile-from-start off` captures this step only
    s0.record()
    step(lev)
    s1.record()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    total = s0.elapsed_time(s1)
    print(f"batch {args.batch} cts ({args.batch * plan.capacity} images): step {total:.2f} ms device, "
          f"{wall * 1e3:.2f} ms wall (unprofiled) -> {args.batch * plan.capacity / wall:.1f} images/s")
    print("per layer (device ms):")
    for name, a, b in lev:
        print(f"  {name:12s} {a.elapsed_time(b):9.3f}")
    print("per C-ABI call:")
    for name, calls, ms in _lib.profile_summary(_lib.PROFILE):
        print(f"  {name:24s} {calls:6d} calls {ms:9.3f} ms  ({100 * ms / total:5.1f}%)")
    if args.trace:
        bounds = marks + [("end", len(_lib.PROFILE))]
        for (name, a), (_, b) in zip(bounds[:-1], bounds[1:]):
            print(f"-- {name}")
            for cname, e0, e1 in _lib.PROFILE[a:b]:
                print(f"     {cname:26s} {e0.elapsed_time(e1):8.3f} ms")
    _lib.PROFILE = None


if __name__ == "__main__":
    main()
