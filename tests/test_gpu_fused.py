"""Fused / hoisted GPU layers vs the op-level schedule, layer by layer.

Both paths run on the GPU backend from the same input state; decrypted
outputs must agree to CKKS rounding (one ModDown + rescale per output instead
of one per product) and the op census of each layer must be identical.
"""

import numpy as np
import pytest

from paper_2402_03060_b200 import driver, fused, planner, schedule
from paper_2402_03060_b200.he_backend import GpuBackend
from paper_2402_03060_b200.params import HEParams
from paper_2402_03060_b200.schedule import CipherState

pytestmark = pytest.mark.gpu


def _dec(be, state):
    return np.stack([np.atleast_2d(be.decrypt(c)) for c in state.cts])


@pytest.mark.parametrize("batch", [1, 3])
def test_layers_fused_equal_oplevel(batch):
    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(seed=5)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    rng = np.random.default_rng(8)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28))) for _ in range(batch)]
    planes = driver.pack_groups(m, groups, plan)
    ct = be.encrypt(be.encode_batch(planes[0]))
    state = schedule.drop_level(be, CipherState([ct], driver._input_layout(m, plan)), 7)
    for layer in m.layers:  # conv, square, pool, conv, square, pool, flatten, fc
        c0 = be.counter.snapshot()
        ref = schedule.apply_layer(be, state, layer)
        c1 = be.counter.snapshot()
        got = fused.apply_layer_fused(be, state, layer)
        c2 = be.counter.snapshot()
        from paper_2402_03060_b200.counter import diff_snapshots

        assert diff_snapshots(c0, c1) == diff_snapshots(c1, c2), type(layer).__name__
        assert got.layout == ref.layout and got.level == ref.level
        a, b = _dec(be, ref), _dec(be, got)
        scale = max(1.0, float(np.max(np.abs(a))))
        assert np.max(np.abs(a - b)) / scale < 1e-7, type(layer).__name__
        state = ref


@pytest.mark.parametrize("name", ["M1", "M6", "M7"])
def test_builtin_models_fused_vs_plaintext(name):
    """Row-removal flatten (M1, M6), conv1d (M7), multi-FC models through the fused path."""
    params = HEParams(poly_degree=1 << 13, depth=8, scale_bits=40)
    m = planner.builtin(name, seed=1)
    # scale the uniform [-0.5, 0.5) weights down so squared activations stay O(1) at 2^40 precision
    for layer in m.layers:
        if hasattr(layer, "weights"):
            layer.weights = layer.weights * 0.2
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    samples = list(np.random.default_rng(2).uniform(0, 1, size=(min(plan.capacity, 4), m.channels, m.height,
                                                                   m.width)))
    outs, metrics, _ = driver.run_inference(m, samples, params, plan=plan, backend=be, fused=True)
    from oracle.slot_sim import SimBackend

    _, ref_metrics, _ = driver.run_inference(m, samples, params, plan=plan, backend=SimBackend(params))
    assert [r.to_dict() for r in metrics.per_layer] == [r.to_dict() for r in ref_metrics.per_layer]
    for s, y in zip(samples, outs):
        ref = planner.reference_infer(m, s)
        assert np.max(np.abs(y - ref)) < 1e-5 * max(1.0, float(np.max(np.abs(ref))))


def test_block_diagonal_hoisted_mac_equals_per_input_sums():
    """uh_hoisted_mac term mode 2 (per-input taps) == the sum of dense single-input calls, residue for residue."""
    import torch

    p = HEParams(poly_degree=1 << 12, depth=3, scale_bits=40, seed=3)
    be = GpuBackend(p)
    level, B, C, R = 2, 3, 3, 2
    rng = np.random.default_rng(7)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, p.num_slots)))) for _ in range(C)]
    X = fused.stack_cts(be, cts, level)  # [C][B][2][L][N]
    shifts = [int(s) for s in rng.integers(-40, 40, size=C * R)]
    rows = rng.uniform(-1, 1, size=(C * R, p.num_slots))
    bank = fused.encode_rows_qp(be, torch.from_numpy(rows).to(be.device), level, float(be.modulus(level)))
    bank = bank.view(1, C * R, level + 2, be.n)
    got = fused._hoist(be, X, level, shifts, bank, 1, 2, B, taps=R)[0]
    want = None
    for i in range(C):
        part = fused._hoist(be, X[i:i + 1].contiguous(), level, shifts[i * R:(i + 1) * R],
                            bank[:, i * R:(i + 1) * R].contiguous(), 1, False, B)[0]
        want = part if want is None else want + part
    mods = [be.modulus(k) for k in range(level + 1)] + [be.modulus(be.sp)]
    q = torch.tensor(mods, dtype=torch.int64, device=be.device).view(1, 1, -1, 1)
    assert torch.equal(got, torch.remainder(want, q))


def test_backend_reused_across_models():
    """One long-lived backend evaluates two models of the same architecture with different
    weights (fused path): the per-layer mask / bias / FC banks are keyed on the layers' content,
    so the second model never picks up the first model's cached banks."""
    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    be = GpuBackend(params)
    rng = np.random.default_rng(30)
    for seed in (40, 41, 40):
        m = planner.lenet1(seed=seed)
        plan = planner.footprint(m, params)
        samples = list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28)))
        outs, _, _ = driver.run_inference(m, samples, params, plan=plan, backend=be, fused=True)
        for y, s in zip(outs, samples):
            assert np.max(np.abs(y - planner.reference_infer(m, s))) < 1e-5


def _census(metrics):
    return [(r.name, r.rotations, r.pt_mults, r.ct_mults, r.adds, r.level_after) for r in metrics.per_layer]


@pytest.mark.parametrize("fused", [False, True], ids=["oplevel", "fused"])
def test_m3_approx_relu_end_to_end(fused):
    """Builtin M3 (conv -> approx_relu -> pool -> flatten -> fc -> approx_relu -> fc, layers.py:238-260
    twice, model.py:676-683) at N = 2^14 on the GPU: decrypted logits within 1e-5 of the plaintext
    forward pass with identical argmax, and the op census / level trace of the reference schedule
    (the slot simulator's) -- the fused approx_relu is one batched masked ct x pt + plaintext add +
    ct x ct + add, with the scale tracked through s -> s^2 / q (the ct + ct adds that follow in
    flatten / fc must not raise ScaleMismatch)."""
    from oracle.slot_sim import SimBackend

    params = HEParams(poly_degree=1 << 14, depth=9, scale_bits=40)
    m = planner.builtin("M3", seed=1)
    plan = planner.footprint(m, params)
    rng = np.random.default_rng(33)
    samples = list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28)))
    be = GpuBackend(params)
    outs, met, _ = driver.run_inference(m, samples, params, plan=plan, backend=be, fused=fused)
    sim = SimBackend(params)
    _, sim_met, _ = driver.run_inference(m, samples, params, plan=plan, backend=sim)
    assert _census(met) == _census(sim_met)
    assert be.counter.by_level == sim.counter.by_level
    for y, s in zip(outs, samples):
        ref = planner.reference_infer(m, s)
        scale = max(1.0, float(np.max(np.abs(ref))))
        assert np.max(np.abs(y - ref)) / scale < 1e-5
        assert int(np.argmax(y)) == int(np.argmax(ref))


def test_approx_relu_fused_equals_oplevel():
    """The fused approx_relu layer equals the op-level schedule on the same input state (3
    ciphertexts, 6 channels, a pending constant from the conv) to CKKS rounding, with the same
    census, level and scale."""
    params = HEParams(poly_degree=1 << 12, depth=9, scale_bits=40)
    m = planner.builtin("M3", seed=2)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    rng = np.random.default_rng(34)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28))) for _ in range(3)]
    planes = driver.pack_groups(m, groups, plan)
    ct = be.encrypt(be.encode_batch(planes[0]))
    state = schedule.drop_level(be, CipherState([ct], driver._input_layout(m, plan)), 9)
    state = fused.apply_layer_fused(be, state, m.layers[0])  # conv: 6 channels
    from paper_2402_03060_b200.counter import diff_snapshots

    c0 = be.counter.snapshot()
    ref = schedule.apply_layer(be, state, m.layers[1])
    c1 = be.counter.snapshot()
    got = fused.apply_layer_fused(be, state, m.layers[1])
    c2 = be.counter.snapshot()
    assert diff_snapshots(c0, c1) == diff_snapshots(c1, c2)
    assert got.layout == ref.layout and got.level == ref.level
    assert all(abs(a.scale - b.scale) <= 1e-9 * a.scale for a, b in zip(got.cts, ref.cts))
    a, b = _dec(be, ref), _dec(be, got)
    assert np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(a)))) < 1e-7
