"""Data parallelism over independent ciphertexts.

The reference is single-process; its only parallelism is SIMD slot packing.
Ciphertexts never exchange data during inference (masks are tiled
identically, layers.py:11-13; the reference's own verification loop already
runs batches independently, engine.py:246-257), so the engine shards the
*ciphertext batch* contiguously across ranks (one process per GPU).  Each
rank derives the evaluation keys from the shared secret seed (zero key
traffic; unseeded parameters would give every rank its own secret, so a
sharded run needs ``HEParams.seed``), encrypts with its own nonce stream, and
the only collective is the final gather of the decrypted logits -- one
fixed-size tensor all-gather over the process group (NCCL over NVLink on GPU
ranks, gloo on CPU ranks).  No data-path collective: weak scaling.
"""

from __future__ import annotations

import math

import numpy as np

from . import driver, planner


def shard_range(n_items: int, rank: int, world: int):
    """Contiguous [start, stop) slice of n_items for rank (sizes differ by at most one)."""
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _out_dim(m) -> int:
    return int(planner.reference_infer(m, np.zeros((m.channels, m.height, m.width))).size)


class _Job:
    """One rank's part of one sharded inference: plan, shard bounds and (packed) host planes."""

    def __init__(self, m, samples, params, backend, group, plan, pinned):
        import torch
        import torch.distributed as dist

        dist_on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if dist_on else 1
        self.rank = dist.get_rank(group) if dist_on else 0
        self.plan = plan or planner.footprint(m, params)
        cap, n = self.plan.capacity, len(samples)
        self.n, self.cap, self.n_groups = n, cap, math.ceil(n / cap)
        self.dout = _out_dim(m)
        self.on_gpu = hasattr(backend, "decrypt_device")
        self.dev = backend.device if self.on_gpu else torch.device("cpu")
        lo, hi = shard_range(self.n_groups, self.rank, self.world)
        mine = [samples[g * cap:min(n, (g + 1) * cap)] for g in range(lo, hi)]
        self.counts = [len(g) for g in mine]
        if (isinstance(samples, np.ndarray) and samples.ndim == 4 and samples.dtype == np.float64 and mine
                and min(self.counts) == cap):
            # full groups of one contiguous array: hand pack_groups the [B, capacity, C, H, W] view
            mine = samples[lo * cap:hi * cap].reshape((hi - lo, cap) + samples.shape[1:])
        self.planes = None
        if len(mine):
            shape = (m.channels, len(mine), self.plan.num_slots)
            if self.on_gpu:
                host = torch.empty(shape, dtype=torch.float64, pin_memory=pinned and torch.cuda.is_available())
                driver.pack_groups(m, mine, self.plan, out=host.numpy())
                self.planes = host
            else:
                self.planes = driver.pack_groups(m, mine, self.plan)

    def enqueue(self, m, params, backend, group, fused):
        """Launch encryption, evaluation, decryption and the logits all-gather; no host sync on
        the GPU path (returns the device tensor of the whole job's logits)."""
        import torch
        import torch.distributed as dist

        local = torch.zeros((0, self.dout), dtype=torch.float64, device=self.dev)
        if self.planes is not None:
            vals, _ = driver.infer_batch(m, self.planes, params, self.plan, backend, counts=self.counts, fused=fused,
                                         as_tensor=True)
            vals = vals.to(self.dev)
            counts = self.counts
            keep = torch.cat([vals[b, :c] for b, c in enumerate(counts)]) if len(counts) > 1 else vals[0, :counts[0]]
            local = keep.reshape(-1, self.dout).contiguous()
        if self.world > 1:
            # per-rank sample counts follow from the deterministic sharding: pad to the largest, gather, trim
            sizes = []
            for r in range(self.world):
                a, b = shard_range(self.n_groups, r, self.world)
                sizes.append(sum(min(self.n, (g + 1) * self.cap) - g * self.cap for g in range(a, b)))
            width = max(sizes)
            buf = torch.zeros((width, self.dout), dtype=torch.float64, device=self.dev)
            buf[:local.shape[0]] = local
            out = torch.empty((self.world * width, self.dout), dtype=torch.float64, device=self.dev)
            dist.all_gather_into_tensor(out, buf, group=group)
            local = torch.cat([out[r * width:r * width + sizes[r]] for r in range(self.world)])
        return local

    def enqueue_to_host(self, m, params, backend, group, fused):
        """``enqueue`` plus an asynchronous device-to-host copy of the logits into pinned memory,
        queued right behind this job's own work; returns (host tensor, completion event or None).
        Waiting on the event waits for this job only -- not for jobs enqueued after it."""
        import torch

        local = self.enqueue(m, params, backend, group, fused)
        if local.device.type != "cuda":
            return local, None
        host = torch.empty(local.shape, dtype=local.dtype, pin_memory=True)
        host.copy_(local, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(local.device))
        return host, ev


def run_sharded(m, samples, params, backend, group=None, fused=True, plan=None, pinned=True):
    """Encrypted inference of ``samples`` sharded over the ranks of ``group``.

    Every rank calls this with the full sample sequence (a list of
    ``(C, H, W)`` arrays or one ``[n, C, H, W]`` array); rank r packs and runs
    the ciphertext groups ``shard_range(groups, r, world)``, then the logits
    of all ranks are gathered so every rank returns the full, ordered
    ``[n, out_dim]`` float64 array.  On a GPU backend the rank's planes are
    packed into pinned host memory (async H2D), its logits stay on the device
    until the NCCL all-gather, and one device-to-host copy ends the call.
    """
    job = _Job(m, samples, params, backend, group, plan, pinned)
    return job.enqueue(m, params, backend, group, fused).cpu().numpy()


def run_sharded_stream(m, batches, params, backend, group=None, fused=True, plan=None, pinned=True):
    """``run_sharded`` over a sequence of sample batches, pipelined: while the GPU evaluates batch
    i, the host packs batch i + 1 into pinned planes and enqueues it, and only then waits for
    batch i's logits -- host packing, H2D and the client-side encode / decrypt overlap the
    evaluation instead of serialising with it.  Yields one ``[n_i, out_dim]`` array per batch
    (same values as ``run_sharded`` on each batch)."""
    it = iter(batches)
    try:
        first = next(it)
    except StopIteration:
        return
    def done(job):
        host, ev = job
        if ev is not None:
            ev.synchronize()  # this batch's D2H only; later batches keep running
        return host.numpy()

    pending = _Job(m, first, params, backend, group, plan, pinned).enqueue_to_host(m, params, backend, group, fused)
    for batch in it:
        nxt = _Job(m, batch, params, backend, group, plan, pinned)  # host packing overlaps the GPU
        queued = nxt.enqueue_to_host(m, params, backend, group, fused)
        yield done(pending)
        pending = queued
    yield done(pending)
