"""Whole-network residue pin of the GPU fused path against the hoisted CPU port.

The same fused layer code (paper_2402_03060_b200.fused) runs once on the GPU kernels and once on
oracle/ckks_hoisted.c (every engine call restated on the host with OpenMP).  With the same keys
(GPU key generation == the oracle's, reproducible mode), the same input ciphertexts and the same
weight-mask banks (the GPU's banks are copied over, so the comparison does not depend on the two
FFT encoders rounding identically at .5 ties), every output residue of the network must be
identical -- this pins the tensor-core conv kernel, the key-bank kernels, the NTT-based ModUp /
ModDown / rescale and the relinearisation at the exact bench shape, not just transitively."""

import numpy as np
import pytest
import torch

from oracle.cpu_backend import CpuHoistedBackend
from paper_2402_03060_b200 import driver, planner
from paper_2402_03060_b200.he_backend import CipherVector, GpuBackend
from paper_2402_03060_b200.params import HEParams
from paper_2402_03060_b200.schedule import CipherState

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("logn,B,tc", [(12, 3, False), (15, 2, False), (15, 2, True)],
                         ids=["N4096", "N32768-mma.sync", "N32768-tcgen05"])
def test_gpu_fused_step_equals_cpu_port(logn, B, tc, monkeypatch):
    monkeypatch.setenv("UH_TC", "1" if tc else "0")
    params = HEParams(poly_degree=1 << logn, depth=9 if logn == 15 else 7, scale_bits=40, seed=11)
    m = planner.lenet1(seed=4)
    plan = planner.footprint(m, params)
    rng = np.random.default_rng(7)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28))) for _ in range(B)]
    planes = driver.pack_groups(m, groups, plan)
    gpu = GpuBackend(params, reproducible=True)
    cts = [gpu.encrypt(gpu.encode_batch(planes[ch])) for ch in range(m.channels)]
    lay = driver._input_layout(m, plan)
    g_state, _, _ = driver._run_layers(m, CipherState(cts, lay), gpu, driver.CostModel(), params.poly_degree, True)
    torch.cuda.synchronize()
    cpu = CpuHoistedBackend(params)
    cpu._mask_banks = {k: v.cpu() for k, v in gpu._mask_banks.items()}
    c_in = [CipherVector(c.data.cpu(), c.level, c.scale, cpu) for c in cts]
    c_state, _, _ = driver._run_layers(m, CipherState(c_in, lay), cpu, driver.CostModel(), params.poly_degree, True)
    assert len(g_state.cts) == len(c_state.cts)
    for g, c in zip(g_state.cts, c_state.cts):
        assert (g.level, g.scale) == (c.level, c.scale)
        assert torch.equal(g.data.cpu(), c.data), "GPU fused step differs from the hoisted CPU port"
    assert gpu.counter.by_level == cpu.counter.by_level
