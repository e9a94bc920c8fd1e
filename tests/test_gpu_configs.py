"""The other BASELINE.json configs as parity cases on the GPU (fused path).

* config 1: Conv 1->4 3x3 -> x^2 -> Flatten -> FC 2704->10 at N=2^14 (depth 4, the
  reference's own depth rule; 3 images per ciphertext) -- exercises 26-tap
  column compaction and a 271-fold FC;
* config 4 (made realisable): CIFAR-shape 3->16 3x3, 16->32 4x4 with
  two pools, FC 1152->10 at N=2^15 (14 images per ciphertext; conv layers wider
  than 12 outputs are split across launches);
* config 5: logistic regression (FC 784->10) and the polynomial-kernel SVM
  (FC 784->256, square, FC 256->1) at N=2^15 with a 60 + 4x40 + 60 chain.

Decrypted outputs vs the plaintext forward pass (north-star tolerance 1e-3,
relative to the output magnitude for the SVM), identical argmax for the
classifiers, and per-layer census identical to the reference schedule.
"""

import numpy as np
import pytest

from oracle.slot_sim import SimBackend
from paper_2402_03060_b200 import driver, planner
from paper_2402_03060_b200.he_backend import GpuBackend
from paper_2402_03060_b200.params import HEParams

pytestmark = pytest.mark.gpu

CASES = {
    "config1": (planner.config1_net, HEParams(poly_degree=1 << 14, depth=4, scale_bits=40)),
    "config4_cifar": (planner.cifar_net, HEParams(poly_degree=1 << 15, depth=9, scale_bits=40)),
    "config5_lr": (planner.lr_model, HEParams(poly_degree=1 << 15, depth=4, scale_bits=40)),
    "config5_svm": (planner.svm_model, HEParams(poly_degree=1 << 15, depth=4, scale_bits=40)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_config_matches_plaintext(name):
    build, params = CASES[name]
    m = build(0)
    plan = planner.footprint(m, params)
    k = min(plan.capacity, 4)
    samples = list(np.random.default_rng(5).uniform(0, 1, size=(k, m.channels, m.height, m.width)))
    be = GpuBackend(params)
    outs, metrics, _ = driver.run_inference(m, samples, params, plan=plan, backend=be, fused=True)
    _, ref_metrics, _ = driver.run_inference(m, samples, params, plan=plan, backend=SimBackend(params))
    assert [r.to_dict() for r in metrics.per_layer] == [r.to_dict() for r in ref_metrics.per_layer]
    for s, y in zip(samples, outs):
        ref = planner.reference_infer(m, s)
        scale = max(1.0, float(np.max(np.abs(ref))))
        assert np.max(np.abs(y - ref)) < 1e-3 * scale
        if ref.size > 1:
            assert np.argmax(y) == np.argmax(ref)
