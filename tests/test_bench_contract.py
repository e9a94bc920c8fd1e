"""The committed round bench line (profiles/r01_bench_b64.json) carries every key of the
bench contract with consistent values (CPU-only: reads the file written on the B200)."""

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    d = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_b64.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["higher_is_better"] is True and d["scaling"] == "weak"
    imgs = d["config"]["ciphertexts_per_gpu_per_step"] * d["config"]["images_per_ciphertext"]
    assert abs(d["value"] - imgs / (d["ms_per_step"] / 1e3)) / d["value"] < 1e-6
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] <= d["value"] * 1.05
    r = d["roofline"]
    assert 0 < r["frac"] <= 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9 and r["traffic"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["value"] > 0
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_mhz"] > 0
    assert d["check"]["argmax_identical"] and d["check"]["max_abs_err_vs_plaintext"] < 1e-3
