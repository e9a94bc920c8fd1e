"""Schedule parity with the reference (no GPU).

* Against the reference package itself (build container only): our schedule,
  planner and driver over the reference's own simulator Backend and over our
  slot restatement reproduce ``slotcnn.run_inference`` bit for bit -- outputs,
  per-layer census rows, totals and level traces -- for M1..M7 and LeNet-1.
* Against the committed golden vectors (everywhere, including the GPU box):
  footprints, capacities, census rows, (kind, level) histograms, level traces,
  simulated outputs and plaintext-oracle outputs recorded from the reference
  by tests/golden/make_golden.py.
"""

import json
import os

import numpy as np
import pytest

from oracle.slot_sim import SimBackend
from paper_2402_03060_b200 import driver, planner
from paper_2402_03060_b200.params import HEParams

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_schedule.json")


def _cases():
    with open(GOLDEN) as fh:
        return json.load(fh)["cases"]


def _model(case):
    return planner.lenet1(0) if case["model"] == "LeNet-1" else planner.builtin(case["model"])


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['model']}-N{c['params']['poly_degree']}")
def test_golden_schedule(case):
    params = HEParams.from_dict(case["params"])
    m = _model(case)
    plan = planner.footprint(m, params)
    assert plan.footprint == case["footprint"] and plan.capacity == case["capacity"]
    samples = np.random.default_rng(case["sample_seed"]).uniform(0.0, 1.0, size=case["samples_shape"])
    be = SimBackend(params)
    outs, metrics, _ = driver.run_inference(m, list(samples), params, plan=plan, backend=be)
    assert [r.level_after for r in metrics.per_layer] == case["level_trace"]
    assert [r.to_dict() for r in metrics.per_layer] == case["rows"]
    assert metrics.totals() == case["totals"]
    assert sorted([[k, lv, c] for (k, lv), c in be.counter.by_level.items()]) == case["hist"]
    for got, want in zip(outs, case["outputs"]):
        assert np.array_equal(got, np.array(want))
    for s, want in zip(samples, case["oracle"]):
        # ours is a plain W @ x in FC; the reference pins the diagonal summation order (model.py:479-506)
        assert np.allclose(planner.reference_infer(m, s), want, rtol=1e-12, atol=1e-12)


def test_golden_m2_census_is_the_survey_census():
    case = [c for c in _cases() if c["model"] == "LeNet-1" and c["params"]["poly_degree"] == 32768][0]
    assert case["capacity"] == 20 and case["footprint"] == 813
    assert case["totals"]["rotations"] == 301 and case["totals"]["pt_mults"] == 1418
    assert case["totals"]["ct_mults"] == 16 and case["level_trace"] == [7, 6, 5, 5, 4, 3, 3, 1, 0]


@pytest.mark.parametrize("name", ["M1", "M2", "M3", "M4", "M5", "M6", "M7", "LeNet-1"])
def test_against_reference_package(reference_slotcnn, name):
    sc = reference_slotcnn
    params = HEParams()
    ref_params = sc.HEParams()
    if name == "LeNet-1":
        from tests.golden.make_golden import lenet1_ref

        rm, mm = lenet1_ref(0), planner.lenet1(0)
    else:
        rm, mm = sc.builtin(name), planner.builtin(name)
    samples = list(np.random.default_rng(9).uniform(0.0, 1.0, size=(3, rm.channels, rm.height, rm.width)))
    r_out, r_met, r_plan = sc.run_inference(rm, samples, ref_params)
    for backend in (sc.Backend(ref_params), SimBackend(params)):
        m_out, m_met, m_plan = driver.run_inference(mm, samples, params, backend=backend)
        assert m_plan.to_dict() == r_plan.to_dict()
        assert all(np.array_equal(a, b) for a, b in zip(r_out, m_out))
        assert [r.to_dict() for r in r_met.per_layer] == [r.to_dict() for r in m_met.per_layer]
        assert [r.detail for r in r_met.per_layer] == [r.detail for r in m_met.per_layer]


def test_reference_engine_over_ckks_backend(reference_slotcnn):
    """Drop-in at the plugin point: the reference's own run_inference (engine.py:196)
    and layers.py, unchanged, drive a real RNS-CKKS backend with our interface."""
    from oracle.ckks_oracle import OracleBackend

    sc = reference_slotcnn
    from tests.golden.make_golden import lenet1_ref

    rm = lenet1_ref(0)
    ref_params = sc.HEParams(poly_degree=1 << 11, depth=7, scale_bits=40)
    be = OracleBackend(HEParams.from_dict(ref_params.to_dict()))
    samples = list(np.random.default_rng(1).uniform(0, 1, size=(1, 1, 28, 28)))  # capacity 1 at N=2^11
    outs, metrics, _ = sc.run_inference(rm, samples, ref_params, backend=be)
    for s, y in zip(samples, outs):
        assert np.max(np.abs(y - sc.reference_infer(rm, s))) < 1e-5
    sim_outs, sim_metrics, _ = sc.run_inference(rm, samples, ref_params)
    assert [r.to_dict() for r in metrics.per_layer] == [r.to_dict() for r in sim_metrics.per_layer]


def test_validation_matches_reference(reference_slotcnn):
    sc = reference_slotcnn
    # config 1 as written (depth 3) fails the reference's depth rule; depth 4 passes
    rng = np.random.default_rng(0)
    w1, b1, w2, b2 = rng.normal(0, .1, (4, 1, 3, 3)), rng.normal(0, .01, 4), rng.normal(0, .05, (10, 2704)), \
        rng.normal(0, .01, 10)
    ref = sc.ModelSpec("c1", 1, 28, 28, (sc.Conv2d(1, 4, 3, 1, w1, b1), sc.Square(), sc.Flatten(),
                                         sc.FC(2704, 10, w2, b2)))
    ours = planner.ModelSpec("c1", 1, 28, 28, (planner.Conv2d(1, 4, 3, 1, w1, b1), planner.Square(),
                                               planner.Flatten(), planner.FC(2704, 10, w2, b2)))
    for depth in (3, 4):
        r = sc.validate(ref, sc.HEParams(poly_degree=1 << 14, depth=depth))
        o = planner.validate(ours, HEParams(poly_degree=1 << 14, depth=depth, scale_bits=40))
        assert (r.ok, r.total_mults, r.per_layer_mults, r.violations) == \
               (o.ok, o.total_mults, o.per_layer_mults, o.violations)


def test_batched_sim_equals_solo():
    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(1)
    plan = planner.footprint(m, params)
    rng = np.random.default_rng(4)
    groups = [list(rng.uniform(0, 1, size=(plan.capacity, 1, 28, 28))) for _ in range(3)]
    outs, metrics = driver.infer_batch(m, driver.pack_groups(m, groups, plan), params, plan, SimBackend(params),
                                       fused=False)
    for b, g in enumerate(groups):
        solo, _, _ = driver.run_inference(m, g, params, plan=plan, backend=SimBackend(params))
        for x, y in zip(outs[b], solo):
            assert np.array_equal(x, y)


def test_pack_groups_fast_path_equals_reference_packing():
    """driver.pack_groups' block-copy path (full groups given as one [B, capacity, C, H, W] array,
    regular offsets) writes exactly planner.batch_pack's layout (packing.py:94-119), into a dirty
    ``out`` buffer too; ragged groups keep the general path."""
    params = HEParams(poly_degree=1 << 13, depth=9, scale_bits=40)
    m = planner.lenet1(0)
    plan = planner.footprint(m, params)
    rng = np.random.default_rng(3)
    B, cap = 3, plan.capacity
    imgs = rng.uniform(0, 1, size=(B * cap, m.channels, m.height, m.width))
    want = np.stack([[pv.values for pv in planner.batch_pack([planner.flatten_input(s) for s in imgs[b * cap:(b + 1) * cap]],
                                                            plan)] for b in range(B)], axis=1)
    out = np.full((m.channels, B, plan.num_slots), 7.0)
    got = driver.pack_groups(m, imgs.reshape(B, cap, m.channels, m.height, m.width), plan, out=out)
    assert got is out and np.array_equal(got, want)
    slow = driver.pack_groups(m, [list(imgs[b * cap:(b + 1) * cap]) for b in range(B)], plan)
    assert np.array_equal(slow, want)
    ragged = driver.pack_groups(m, [imgs[:cap], imgs[cap:cap + 2]], plan)
    assert np.array_equal(ragged[:, 0], want[:, 0]) and not ragged[:, 1, plan.offsets[2]:].any()
