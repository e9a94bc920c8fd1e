"""The committed bench lines (profiles/r01_bench_b64.json, profiles/r02_bench_b128.json) carry every
key of the bench contract with consistent values (CPU-only: reads the files written on the B200),
and -- on a GPU box -- bench.py's multi-rank path runs end to end under torchrun."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["r01_bench_b64.json", "r02_bench_b128.json"])
def test_bench_line_contract(name):
    d = json.load(open(os.path.join(ROOT, "profiles", name)))
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
    assert c["kind"] in ("port", "port-hoisted", "reference") and c["cores"] >= 1 and c["value"] > 0
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_mhz"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert d["check"]["argmax_identical"] and d["check"]["max_abs_err_vs_plaintext"] < 1e-3


@pytest.mark.gpu
def test_bench_two_ranks_under_torchrun(tmp_path):
    """bench.py under torchrun with 2 ranks -- the launch the driver uses for the scaling run --
    as a functional smoke on one GPU (UH_BENCH_DIST_BACKEND=gloo: both ranks on cuda:0, host-side
    collectives): rank 0 prints one line with n_gpus 2, the whole-job value, and an e2e check of
    every image of both ranks' shards against the plaintext forward pass."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, UH_BENCH_DIST_BACKEND="gloo", OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--batch", "4", "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 2 * 4 * 20
    assert abs(d["value"] - 2 * 4 * 20 / (d["ms_per_step"] / 1e3)) / d["value"] < 1e-6
    chk = d["e2e"]["check"]
    assert chk["images_checked"] == 2 * 4 * 20 and chk["argmax_identical"]
    assert chk["max_abs_err_vs_plaintext"] < 1e-3
