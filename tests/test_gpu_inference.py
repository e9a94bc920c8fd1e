"""End-to-end encrypted inference on the GPU backend.

Decrypted logits vs the plaintext forward pass (tolerance 1e-3 absolute as
the north star states; the achieved error is asserted far tighter), argmax
agreement, and an op census / level trace identical to the reference
schedule's (run here over the slot restatement, pinned to the reference by
tests/golden/).
"""

import numpy as np
import pytest

from oracle.slot_sim import SimBackend
from paper_2402_03060_b200 import driver, planner
from paper_2402_03060_b200.he_backend import GpuBackend
from paper_2402_03060_b200.params import HEParams

pytestmark = pytest.mark.gpu

TOL = 1e-3  # north star: decrypted logits within 1e-3 absolute
M2_TRACE = [7, 6, 5, 5, 4, 3, 3, 1, 0]


def _samples(m, k, seed):
    return list(np.random.default_rng(seed).uniform(0.0, 1.0, size=(k, m.channels, m.height, m.width)))


@pytest.mark.parametrize("fused", [False, True], ids=["oplevel", "fused"])
@pytest.mark.parametrize("params", [HEParams(poly_degree=1 << 12, depth=7, scale_bits=40),
                                    HEParams(poly_degree=1 << 15, depth=9, scale_bits=40)],
                         ids=lambda p: f"N{p.poly_degree}")
def test_lenet1_matches_plaintext(params, fused):
    m = planner.lenet1(seed=0)
    plan = planner.footprint(m, params)
    samples = _samples(m, plan.capacity, seed=1)
    be = GpuBackend(params)
    outs, metrics, _ = driver.run_inference(m, samples, params, plan=plan, backend=be, fused=fused)
    errs = []
    for s, y in zip(samples, outs):
        ref = planner.reference_infer(m, s)
        errs.append(float(np.max(np.abs(y - ref))))
        assert np.argmax(y) == np.argmax(ref)
    assert max(errs) < TOL
    assert max(errs) < 1e-5, f"CKKS error {max(errs):.3e} larger than expected"
    assert [r.level_after for r in metrics.per_layer] == M2_TRACE
    sim = SimBackend(params)
    _, sim_metrics, _ = driver.run_inference(m, samples, params, plan=plan, backend=sim)
    assert metrics.totals() == sim_metrics.totals()
    assert be.counter.by_level == sim.counter.by_level


def test_batched_equals_solo_within_tolerance():
    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(seed=2)
    plan = planner.footprint(m, params)
    groups = [_samples(m, plan.capacity, seed=10 + b) for b in range(3)]
    be = GpuBackend(params)
    planes = driver.pack_groups(m, groups, plan)
    outs, metrics = driver.infer_batch(m, planes, params, plan, be, fused=True)
    for b, group in enumerate(groups):
        for s, y in zip(group, outs[b]):
            assert np.max(np.abs(y - planner.reference_infer(m, s))) < 1e-5
    assert [r.level_after for r in metrics.per_layer] == M2_TRACE


def test_pinned_tensor_client_path_matches_numpy_path():
    """driver.infer_batch with pinned float64 planes (GpuBackend.encrypt_slots, async H2D) gives the
    same logits as the numpy path (ciphertext ids continue, so the noise differs: compare to 1e-5)."""
    import torch

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(seed=3)
    plan = planner.footprint(m, params)
    groups = [_samples(m, plan.capacity, seed=20 + b) for b in range(2)]
    planes = driver.pack_groups(m, groups, plan)
    be = GpuBackend(params)
    a, _ = driver.infer_batch(m, planes, params, plan, be, fused=True)
    b, _ = driver.infer_batch(m, torch.from_numpy(np.ascontiguousarray(planes)).pin_memory(), params, plan, be,
                              fused=True)
    for ga, gb, group in zip(a, b, groups):
        for ya, yb, s in zip(ga, gb, group):
            ref = planner.reference_infer(m, s)
            assert np.max(np.abs(ya - ref)) < 1e-5 and np.max(np.abs(yb - ref)) < 1e-5


def test_encrypt_slots_rules():
    import torch

    from paper_2402_03060_b200.errors import OversizedInput

    params = HEParams(poly_degree=64, depth=2, scale_bits=40)
    be = GpuBackend(params)
    x = torch.linspace(-1, 1, 10, dtype=torch.float64).view(1, 10)
    c = be.encrypt_slots(x)
    d = be.decrypt(c)
    assert np.max(np.abs(d[:10] - x.numpy()[0])) < 1e-6 and np.max(np.abs(d[10:])) < 1e-6
    with pytest.raises(OversizedInput):
        be.encrypt_slots(torch.zeros((1, params.num_slots + 1), dtype=torch.float64))
    with pytest.raises(OversizedInput):
        be.encrypt_slots(torch.zeros(5, dtype=torch.float64))


def test_throughput_config_40960_images():
    """The realisable throughput configuration (config-2 network, 20 images per
    ciphertext x 2048 ciphertexts = 40,960 images) in B = 64 chunks through driver.infer_batch:
    every image's decrypted logits against the plaintext forward pass (engine.py:233-265 style
    argmax agreement).  Any argmax flip must be an image whose plaintext top-2 gap is below twice
    the achieved error (a near tie); the committed artifact of the same run is
    profiles/r02_parity_40960.json."""
    import importlib.util
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts",
                        "parity_throughput.py")
    spec = importlib.util.spec_from_file_location("parity_throughput", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    res = mod.run(n_ct=2048, batch=64)
    assert res["images"] == 40960
    assert res["max_abs_err"] < 1e-5  # north star 1e-3; achieved ~1e-6
    for f in res["argmax_flips"]:
        assert f["ref_top2_gap"] < 2 * res["max_abs_err"], f
    assert res["argmax_agreement"] >= 1.0 - len(res["near_ties_below_2x_max_err"]) / 40960


@pytest.mark.parametrize("logn", [12, 15])
def test_graph_replayed_step_equals_eager(logn):
    """driver.EvalGraph: the whole fused LeNet-1 evaluation captured as one CUDA graph; replays on two
    different input batches give residues identical to eager runs, and decrypt to the plaintext."""
    import torch

    from paper_2402_03060_b200.schedule import CipherState

    params = HEParams(poly_degree=1 << logn, depth=9 if logn == 15 else 7, scale_bits=40)
    m = planner.lenet1(seed=3)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    B = 3
    g = driver.EvalGraph(m, plan, be, B)
    for seed in (20, 21):
        groups = [_samples(m, plan.capacity, seed=seed * 10 + b) for b in range(B)]
        planes = driver.pack_groups(m, groups, plan)
        cts = [be.encrypt(be.encode_batch(planes[ch])) for ch in range(m.channels)]
        outs = g.run(cts)
        torch.cuda.synchronize()
        got = [c.data.clone() for c in outs]
        state, _, _ = driver._run_layers(m, CipherState(cts, driver._input_layout(m, plan)), be, driver.CostModel(),
                                         params.poly_degree, True)
        for a, c in zip(got, state.cts):
            assert torch.equal(a, c.data)
        lay = state.layout
        pos = driver.valid_positions(lay)
        dec = [np.atleast_2d(be.decrypt(c)) for c in outs]
        for b in range(B):
            for i, off in enumerate(plan.offsets[:plan.capacity]):
                y = np.concatenate([d[b][off + pos] for d in dec]) * lay.pending_const
                ref = planner.reference_infer(m, groups[b][i])
                assert np.max(np.abs(y - ref)) < 1e-5


def test_stream_on_gpu_equals_per_batch_runs():
    """shard.run_sharded_stream on GpuBackend (pinned planes, async D2H per batch) returns what
    run_sharded returns for each batch, within CKKS noise (fresh encryption nonces per call)."""
    from paper_2402_03060_b200.shard import run_sharded, run_sharded_stream

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(seed=6)
    be = GpuBackend(params)
    rng = np.random.default_rng(31)
    batches = [rng.uniform(0, 1, size=(k, 1, 28, 28)) for k in (5, 2, 3)]
    streamed = list(run_sharded_stream(m, batches, params, be))
    for b, got in zip(batches, streamed):
        want = run_sharded(m, b, params, be)
        assert got.shape == want.shape == (len(b), 10)
        assert np.max(np.abs(got - want)) < 1e-5
        for i in range(len(b)):
            assert np.max(np.abs(got[i] - planner.reference_infer(m, b[i]))) < 1e-5


def test_eval_graph_rejects_other_shapes():
    from paper_2402_03060_b200.errors import ShapeMismatch

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(seed=3)
    plan = planner.footprint(m, params)
    be = GpuBackend(params)
    g = driver.EvalGraph(m, plan, be, 2)
    planes = driver.pack_groups(m, [_samples(m, plan.capacity, seed=1)] * 3, plan)
    cts = [be.encrypt(be.encode_batch(planes[ch])) for ch in range(m.channels)]  # 3 ciphertexts, not 2
    with pytest.raises(ShapeMismatch):
        g.run(cts)
    with pytest.raises(ShapeMismatch):
        g.run([])
