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
    import torch
    import torch.distributed as dist

    dist_on = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if dist_on else 1
    rank = dist.get_rank(group) if dist_on else 0
    if plan is None:
        plan = planner.footprint(m, params)
    cap, n = plan.capacity, len(samples)
    n_groups = math.ceil(n / cap)
    dout = _out_dim(m)
    on_gpu = hasattr(backend, "decrypt_device")
    dev = backend.device if on_gpu else torch.device("cpu")
    lo, hi = shard_range(n_groups, rank, world)
    mine = [samples[g * cap:min(n, (g + 1) * cap)] for g in range(lo, hi)]
    counts = [len(g) for g in mine]
    local = torch.zeros((0, dout), dtype=torch.float64, device=dev)
    if mine:
        shape = (m.channels, len(mine), plan.num_slots)
        if on_gpu:
            host = torch.empty(shape, dtype=torch.float64, pin_memory=pinned and torch.cuda.is_available())
            driver.pack_groups(m, mine, plan, out=host.numpy())
            planes = host
        else:
            planes = driver.pack_groups(m, mine, plan)
        vals, _ = driver.infer_batch(m, planes, params, plan, backend, counts=counts, fused=fused, as_tensor=True)
        vals = vals.to(dev)
        keep = torch.cat([vals[b, :c] for b, c in enumerate(counts)]) if len(counts) > 1 else vals[0, :counts[0]]
        local = keep.reshape(-1, dout).contiguous()
    if world > 1:
        # per-rank sample counts follow from the deterministic sharding: pad to the largest, gather, trim
        sizes = []
        for r in range(world):
            a, b = shard_range(n_groups, r, world)
            sizes.append(sum(min(n, (g + 1) * cap) - g * cap for g in range(a, b)))
        width = max(sizes)
        buf = torch.zeros((width, dout), dtype=torch.float64, device=dev)
        buf[:local.shape[0]] = local
        out = torch.empty((world * width, dout), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(out, buf, group=group)
        local = torch.cat([out[r * width:r * width + sizes[r]] for r in range(world)])
    return local.cpu().numpy()
