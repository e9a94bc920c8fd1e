"""ctypes binding of the C-ABI in ``include/unihenn_b200.h``.

The shared library is built in-tree (``paper_2402_03060_b200/_build``) by
:func:`paper_2402_03060_b200.build.build`.  There is no fallback: if the
library is missing or fails to load, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError

LIB_NAME = "libunihenn_b200.so"
LIB_PATH = os.environ.get("UH_LIB_PATH") or os.path.join(  # override: A/B builds of compile-time variants
    os.path.dirname(os.path.abspath(__file__)), "_build", LIB_NAME)

_c_u32, _c_u64, _c_i64, _c_int, _c_dbl, _vp = (ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int,
                                               ctypes.c_double, ctypes.c_void_p)

# name -> argtypes (all return int status except the two noted)
SIGNATURES = {
    "uh_ctx_create": [ctypes.POINTER(_vp), _c_u32, _vp, _vp, _c_u32, _c_int],
    "uh_ctx_destroy": [_vp],
    "uh_ntt": [_vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_elementwise": [_vp, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_elementwise_grouped": [_vp, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                               _c_int, _vp],
    "uh_divide_top": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_rescale": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_divide_top2": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_divide_top2_bias": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "uh_modup": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp],
    "uh_key_inner": [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_i64, _vp],
    "uh_keyswitch": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "uh_rotate": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_i64, _vp],
    "uh_rotate_hoisted": [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_i64, _vp],
    "uh_mul_plain_rescale": [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_mul_relin_rescale": [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "uh_mul_relin_rescale_fused": [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "uh_secret_gen": [_vp, _vp, _c_u64, _vp],
    "uh_galois_keygen": [_vp, _vp, _vp, _c_u64, _c_i64, _c_int, _vp],
    "uh_relin_keygen": [_vp, _vp, _vp, _c_u64, _c_int, _vp],
    "uh_encrypt": [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_u64, _c_u64, _vp],
    "uh_decrypt_coeffs": [_vp, _vp, _vp, _vp, _c_int, _c_int, _vp],
    "uh_encode_coeffs": [_vp, _vp, _vp, _c_int, _c_dbl, _vp],
    "uh_from_signed": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp],
    "uh_decode_coeffs": [_vp, _vp, _vp, _c_int, _c_dbl, _vp],
    "uh_from_signed_qp": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp],
    "uh_conv_hoisted_mac": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int,
                            _c_int, _vp],
    "uh_rot_sum_hoisted": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_hoisted_mac": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                       _vp],
    "uh_hoisted_mac_bank": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                            _vp],
    "uh_km_bank": [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_hoisted_mac_km": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_imma_ta_bank": [_vp, _vp, _vp, _vp, _c_int, _c_int, _vp],
    "uh_hoisted_mac_imma_ta": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int,
                               _vp],
    "uh_imma_mask_bank": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp],
    "uh_tc_mask_bank": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp],
    "uh_hoisted_mac_tc": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp],
    "uh_hoisted_mac_imma": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int,
                            _vp],
}
EXTRA = {"uh_abi_version": ([], _c_int), "uh_last_error": ([], ctypes.c_char_p),
         "uh_launch_count": ([], ctypes.c_ulonglong), "uh_bench_peaks": ([_vp, _vp], _c_int),
         "uh_hoisted_bank_supported": ([_vp, _c_int, _c_int], _c_int),
         "uh_km_supported": ([_vp, _c_int], _c_int),
         "uh_divide_top2_bias_supported": ([_vp], _c_int),
         "uh_imma_supported": ([_vp, _c_int, _c_int, _c_int], _c_int),
         "uh_imma_ta_supported": ([_vp, _c_int, _c_int, _c_int], _c_int),
         "uh_imma_ta_bank_bytes": ([_vp, _c_int, _c_int], ctypes.c_ulonglong),
         "uh_imma_bank_words": ([_vp, _c_int, _c_int, _c_int], ctypes.c_ulonglong),
         "uh_tc_supported": ([_vp, _c_int, _c_int, _c_int], _c_int),
         "uh_tc_bank_bytes": ([_vp, _c_int, _c_int, _c_int], ctypes.c_ulonglong)}


def launch_count() -> int:
    return int(load().uh_launch_count())

_LIB = None


def load():
    """Load the engine library (no compute happens here)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"CUDA engine library missing: {LIB_PATH} (run __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _c_int
        for name, (args, res) in EXTRA.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = lib
    return _LIB


PROFILE = None  # set to a list to record (name, start_event, end_event) around every call


def call(name: str, *args) -> None:
    lib = load()
    if PROFILE is not None:
        import torch

        s = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        rc = getattr(lib, name)(*args)
        e1.record(s)
        PROFILE.append((name, e0, e1))
    else:
        rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.uh_last_error().decode(errors="replace")
        raise DeviceError(f"{name}: {msg}")


def profile_summary(records) -> list:
    """[(name, calls, total_ms)] sorted by total time (events must be complete)."""
    agg = {}
    for name, e0, e1 in records:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += e0.elapsed_time(e1)
    return sorted(((k, v[0], v[1]) for k, v in agg.items()), key=lambda x: -x[2])
