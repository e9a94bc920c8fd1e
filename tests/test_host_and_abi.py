"""Host-side logic and the C-ABI boundary (no GPU needed).

* the engine library loads and exports every symbol include/unihenn_b200.h declares
  (no compute call is made without a GPU);
* HEParams keeps the reference's validation and dict round trip
  (he_backend.py:34-77; tests/test_he_backend.py:16-45 of the reference);
* GpuBackend fails loudly without a device (no CPU fallback);
* planner footprints / capacities equal the reference's (test_packing.py:21-22);
* the op counter / diff_snapshots contract (he_backend.py:104-152).
"""

import os
import re

import pytest

from paper_2402_03060_b200 import _lib, planner
from paper_2402_03060_b200.counter import OpCounter, diff_snapshots
from paper_2402_03060_b200.errors import DeviceError
from paper_2402_03060_b200.params import HEParams

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "unihenn_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(uh_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.uh_abi_version() == 1
    # every declared entry point has a ctypes signature in the binding
    assert set(syms) <= set(_lib.SIGNATURES) | set(_lib.EXTRA)


def test_null_context_reports_error_not_crash():
    import ctypes

    with pytest.raises(DeviceError, match="null context"):
        _lib.call("uh_ntt", ctypes.c_void_p(0), ctypes.c_void_p(0), 1, 1, 1, 1, 0, ctypes.c_void_p(0))


def test_params_validation_matches_reference():
    for bad in (0, 3, 6, 12, 1000):
        with pytest.raises(ValueError):
            HEParams(poly_degree=bad)
    with pytest.raises(ValueError):
        HEParams(depth=0)
    with pytest.raises(ValueError):
        HEParams(scale_bits=0)
    with pytest.raises(ValueError):
        HEParams(log_q=0)
    p = HEParams(poly_degree=4096, depth=9, scale_bits=20, quantize=True, log_q=100)
    assert HEParams.from_dict(p.to_dict()) == p
    assert HEParams.from_dict({"poly_degree": 64, "unknown": 1}).poly_degree == 64
    assert HEParams().num_slots == 8192


def test_gpu_backend_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2402_03060_b200.he_backend import GpuBackend

    with pytest.raises(DeviceError):
        GpuBackend(HEParams(poly_degree=64, depth=2, scale_bits=40))


FOOTPRINTS = {"M1": 784, "M2": 813, "M3": 1080, "M4": 1057, "M5": 1123, "M6": 320, "M7": 128}  # reference values


@pytest.mark.parametrize("name", sorted(FOOTPRINTS))
def test_planner_footprints(name):
    plan = planner.footprint(planner.builtin(name), HEParams())
    assert plan.footprint == FOOTPRINTS[name]
    assert plan.capacity == HEParams().num_slots // FOOTPRINTS[name]


def test_counter_contract():
    c = OpCounter()
    before = c.snapshot()
    c.record("rotation", 2)
    c.record("rotation", 2)
    c.record("add", 1)
    c.record("pt_mult", 3, count=4)
    totals, hist = diff_snapshots(before, c.snapshot())
    assert totals == {"rotations": 2, "pt_mults": 4, "ct_mults": 0, "adds": 1}
    assert hist == {("rotation", 2): 2, ("add", 1): 1, ("pt_mult", 3): 4}
