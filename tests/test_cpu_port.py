"""The hoisted CPU port (oracle/ckks_hoisted.c behind oracle/cpu_backend.py): the unchanged fused
layer path on the host.  CPU-only checks; the GPU == port residue comparison is
tests/test_gpu_cpu_port.py."""

import numpy as np
import pytest

from oracle.cpu_backend import CpuHoistedBackend
from paper_2402_03060_b200 import driver, planner
from paper_2402_03060_b200.params import HEParams


def test_cpu_port_lenet1_matches_plaintext():
    """Fused LeNet-1 (every layer hoisted: conv, square, pool, flatten, FC) on the CPU port at
    N = 2^12, two ciphertexts, decrypts to the plaintext forward pass with identical argmax."""
    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40, seed=5)
    m = planner.lenet1(seed=0)
    plan = planner.footprint(m, params)
    rng = np.random.default_rng(1)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28))) for _ in range(2)]
    be = CpuHoistedBackend(params)
    outs, metrics = driver.infer_batch(m, driver.pack_groups(m, groups, plan), params, plan, be, fused=True)
    for b in range(2):
        for i in range(plan.capacity):
            ref = planner.reference_infer(m, groups[b][i])
            assert np.max(np.abs(outs[b][i] - ref)) < 1e-5
            assert np.argmax(outs[b][i]) == np.argmax(ref)


def test_cpu_port_needs_seed():
    with pytest.raises(ValueError):
        CpuHoistedBackend(HEParams(poly_degree=1 << 12, depth=7, scale_bits=40))
