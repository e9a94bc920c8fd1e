"""Generate golden vectors from the REFERENCE package (run in the build container).

    python tests/golden/make_golden.py

Imports ``slotcnn`` from /root/reference/pkg/src (read-only) and records, per
model and parameter set, what the reference's own schedule and oracle produce:
footprint/capacity, per-layer census rows, the (kind, level) histogram, level
traces, the decrypted (simulated) outputs of seeded samples and the plaintext
oracle outputs.  The committed JSON lets the GPU box (no reference there)
check the engine's schedule, census and decrypted logits against the
reference.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import slotcnn  # noqa: E402


def lenet1_ref(seed=0):
    """BASELINE config-2 network in the reference's own types (same draws as planner.lenet1)."""
    rng = np.random.default_rng(seed)
    w = lambda *s: rng.normal(0.0, 0.1, size=s)  # noqa: E731
    b = lambda *s: rng.normal(0.0, 0.01, size=s)  # noqa: E731
    layers = []
    c1w = w(4, 1, 5, 5)
    layers.append(slotcnn.Conv2d(1, 4, 5, 1, c1w, b(4)))
    layers.append(slotcnn.Square())
    layers.append(slotcnn.AvgPool2d(2))
    c2w = w(12, 4, 5, 5)
    layers.append(slotcnn.Conv2d(4, 12, 5, 1, c2w, b(12)))
    layers.append(slotcnn.Square())
    layers.append(slotcnn.AvgPool2d(2))
    layers.append(slotcnn.Flatten())
    fw = w(10, 192)
    layers.append(slotcnn.FC(192, 10, fw, b(10)))
    return slotcnn.ModelSpec("LeNet-1", 1, 28, 28, tuple(layers))


def record(name, m, params, n_samples=2, seed=3):
    plan = slotcnn.footprint(m, params)
    k = min(n_samples, plan.capacity)
    rng = np.random.default_rng(seed)
    samples = rng.uniform(0.0, 1.0, size=(k, m.channels, m.height, m.width))
    be = slotcnn.Backend(params)
    outs, metrics, _ = slotcnn.run_inference(m, list(samples), params, plan=plan, backend=be)
    return {
        "model": name,
        "params": params.to_dict(),
        "footprint": plan.footprint,
        "capacity": plan.capacity,
        "level_trace": [r.level_after for r in metrics.per_layer],
        "rows": [r.to_dict() for r in metrics.per_layer],
        "totals": metrics.totals(),
        "hist": sorted([[kind, lvl, cnt] for (kind, lvl), cnt in be.counter.by_level.items()]),
        "sample_seed": seed,
        "samples_shape": list(samples.shape),
        "outputs": [o.tolist() for o in outs],
        "oracle": [slotcnn.reference_infer(m, s).tolist() for s in samples],
    }


def main():
    out = []
    default = slotcnn.HEParams()
    for name in slotcnn.builtin_names():
        out.append(record(name, slotcnn.builtin(name), default))
    c2 = slotcnn.HEParams(poly_degree=1 << 15, depth=9, scale_bits=40)
    out.append(record("LeNet-1", lenet1_ref(0), c2, n_samples=20))
    small = slotcnn.HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    out.append(record("LeNet-1", lenet1_ref(0), small, n_samples=2))
    path = os.path.join(HERE, "reference_schedule.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "slotcnn 0.1.0 (/root/reference/pkg)",
                   "cases": out}, fh, indent=0)
    print(path, len(out), "cases")


if __name__ == "__main__":
    main()
