"""Integer- and FP64-pipe peaks of this GPU (uh_bench_peaks)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_03060_b200 import _lib  # noqa: E402
from paper_2402_03060_b200.he_backend import GpuBackend  # noqa: E402
from paper_2402_03060_b200.params import HEParams  # noqa: E402

NAMES = ["IMAD", "MAC128 (engine, IMAD.WIDE chain)", "mulmod (reduced)", "MAC128 (plain-C form)",
         "Shoup lazy", "FP64 exact modMAC (q<2^50)", "mixed IMAD+FP64 MAC", "MAC128 split accumulator (AccS)",
         "narrow-operand MAC (AccN, q < 2^41)", "u8 IMMA MAC (mma.sync m16n8k32)", "FP64 FMA",
         "tcgen05 kind::i8 MAC (M128 N256 K32)", "split-FP64 MAC (q < 2^40, one operand split per MAC)",
         "split-FP64 MAC (both operands pre-split: 4 DFMA)"]

if __name__ == "__main__":
    be = GpuBackend(HEParams(poly_degree=1 << 12, depth=2, scale_bits=40))
    r = np.zeros(16)
    _lib.call("uh_bench_peaks", be._ctx, ctypes.c_void_p(r.ctypes.data))
    for name, v in zip(NAMES, r):
        print(f"{name:36s} {v / 1e12:8.3f} T/s")
