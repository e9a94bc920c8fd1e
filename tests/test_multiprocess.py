"""Multi-rank path on CPU: world_size 2 over gloo (127.0.0.1).

The ciphertext batch is sharded contiguously across ranks with no data-path
collective; only the decrypted logits are gathered.  Each rank runs the real
schedule (over the batch-aware slot restatement on CPU); the gathered result
must equal a single-process run sample for sample, in order.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_03060_b200 import driver, planner
from paper_2402_03060_b200.params import HEParams
from paper_2402_03060_b200.shard import run_sharded, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_samples, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.slot_sim import SimBackend

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(3)
    samples = list(np.random.default_rng(11).uniform(0, 1, size=(n_samples, 1, 28, 28)))
    outs = run_sharded(m, samples, params, SimBackend(params), fused=False)
    if rank == 0:
        np.save(out_path, np.stack(outs))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 5, 7, 64):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


@pytest.mark.parametrize("n_samples", [7, 1])  # 1: rank 1 owns no group
def test_two_rank_gloo_equals_single_process(tmp_path, n_samples):
    out = str(tmp_path / "outs.npy")
    mp.spawn(_worker, args=(2, _free_port(), n_samples, out), nprocs=2, join=True)
    got = np.load(out)
    from oracle.slot_sim import SimBackend

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40)
    m = planner.lenet1(3)
    samples = list(np.random.default_rng(11).uniform(0, 1, size=(n_samples, 1, 28, 28)))
    plan = planner.footprint(m, params)
    want = []
    for i in range(0, n_samples, plan.capacity):
        o, _, _ = driver.run_inference(m, samples[i:i + plan.capacity], params, plan=plan,
                                       backend=SimBackend(params))
        want.extend(o)
    assert got.shape == (n_samples, 10)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def _gpu_worker(rank, world, port, n_samples, out_path):
    """One rank of the GPU sharded path; both ranks share cuda:0 (independent work, no
    cross-rank waits inside kernels), logits gathered over gloo on host tensors."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_03060_b200.he_backend import GpuBackend

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40, seed=21)
    m = planner.lenet1(4)
    samples = np.random.default_rng(12).uniform(0, 1, size=(n_samples, 1, 28, 28))
    be = GpuBackend(params)
    import torch

    got = run_sharded(m, samples, params, be, fused=True)
    if rank == 0:
        np.save(out_path, got)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_backend_equals_single_process(tmp_path):
    """world_size 2 on one GPU: GpuBackend per rank (keys from the shared secret seed, own nonce
    streams), fused layers, logits gathered through the tensor all-gather -- equal to a
    single-process sharded run and to the plaintext forward pass within CKKS tolerance."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n_samples = 9  # 5 ciphertext groups of capacity 2: ranks own 3 and 2
    out = str(tmp_path / "outs.npy")
    mp.spawn(_gpu_worker, args=(2, _free_port(), n_samples, out), nprocs=2, join=True)
    got = np.load(out)
    from paper_2402_03060_b200.he_backend import GpuBackend

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40, seed=21)
    m = planner.lenet1(4)
    samples = np.random.default_rng(12).uniform(0, 1, size=(n_samples, 1, 28, 28))
    single = run_sharded(m, samples, params, GpuBackend(params), fused=True)
    assert got.shape == single.shape == (n_samples, 10)
    ref = np.stack([planner.reference_infer(m, s) for s in samples])
    assert np.max(np.abs(got - single)) < 1e-5
    assert np.max(np.abs(got - ref)) < 1e-5
    assert np.array_equal(np.argmax(got, 1), np.argmax(ref, 1))


def test_stream_equals_per_batch_runs():
    """run_sharded_stream (host packing of batch i + 1 overlapped with batch i) returns, batch for
    batch, what run_sharded returns -- on the hoisted CPU port (the fused path, real CKKS)."""
    from oracle.cpu_backend import CpuHoistedBackend
    from paper_2402_03060_b200.shard import run_sharded_stream

    params = HEParams(poly_degree=1 << 12, depth=7, scale_bits=40, seed=9)
    m = planner.lenet1(5)
    rng = np.random.default_rng(12)
    batches = [rng.uniform(0, 1, size=(k, 1, 28, 28)) for k in (3, 1, 2)]
    be = CpuHoistedBackend(params)
    streamed = list(run_sharded_stream(m, batches, params, be))
    assert len(streamed) == len(batches)
    for b, got in zip(batches, streamed):
        want = run_sharded(m, b, params, be)
        assert got.shape == want.shape
        assert np.allclose(got, want, atol=1e-6)
        for i in range(len(b)):
            assert np.max(np.abs(got[i] - planner.reference_infer(m, b[i]))) < 1e-5
