"""Throughput of the NTT-based primitives at N=2^15 (device time, CUDA events)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_03060_b200 import _lib  # noqa: E402
from paper_2402_03060_b200.he_backend import GpuBackend  # noqa: E402
from paper_2402_03060_b200.params import HEParams  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    if "--ncu" in sys.argv:  # one call of each primitive inside cudaProfilerStart/Stop (ncu --profile-from-start off)
        global timeit

        def timeit(fn, reps=5):
            fn()
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
            fn()
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            return 1.0
    p = HEParams(poly_degree=1 << 15, depth=9, scale_bits=40)
    be = GpuBackend(p)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    n = p.poly_degree
    polys, nl = 64, 8
    x = torch.randint(0, 1 << 39, (polys, nl, n), dtype=torch.int64, device="cuda")
    limbs = polys * nl
    for inv in (0, 1):
        ms = timeit(lambda: _lib.call("uh_ntt", be._ctx, vp(x), polys, nl, nl, nl, inv, st))
        print(f"{'inverse' if inv else 'forward'} NTT: {limbs} limbs {ms:.3f} ms -> {1e3 * ms / limbs:.3f} us/limb, "
              f"{limbs * n * 16 / (ms * 1e-3) / 1e9:.0f} GB/s (r+w)")
    # 60-bit limbs only (q_0: nl = nq = 1) vs the mixed 8-limb case above (1 x 60-bit + 7 x 40-bit)
    x1 = torch.randint(0, 1 << 39, (limbs, 1, n), dtype=torch.int64, device="cuda")
    ms = timeit(lambda: _lib.call("uh_ntt", be._ctx, vp(x1), limbs, 1, 1, 1, 0, st))
    print(f"forward NTT, 60-bit q_0 limbs only: {limbs} limbs -> {1e3 * ms / limbs:.3f} us/limb")
    lev = 5
    L = lev + 1
    d = torch.randint(0, 1 << 39, (polys, L, n), dtype=torch.int64, device="cuda")
    D = torch.empty((polys, L, L + 1, n), dtype=torch.int64, device="cuda")
    ms = timeit(lambda: _lib.call("uh_modup", be._ctx, vp(D), vp(d), polys, lev, L, st))
    nt = polys * (L + L * (L + 1))
    print(f"modup level {lev}: {polys} polys {ms:.3f} ms ({nt} limb-NTTs -> {1e3 * ms / nt:.3f} us/limb-NTT)")
    u = torch.randint(0, 1 << 39, (polys, L + 1, n), dtype=torch.int64, device="cuda")
    out = torch.empty((polys, L, n), dtype=torch.int64, device="cuda")
    ms = timeit(lambda: _lib.call("uh_divide_top", be._ctx, vp(out), vp(u), polys, L, be.sp, L, L + 1, st))
    nt = polys * (1 + L)
    print(f"moddown level {lev}: {polys} polys {ms:.3f} ms ({nt} limb-NTTs -> {1e3 * ms / nt:.3f} us/limb-NTT)")


if __name__ == "__main__":
    main()
