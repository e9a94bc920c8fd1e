"""Data parallelism over independent ciphertexts.

The reference is single-process; its only parallelism is SIMD slot packing.
Ciphertexts never exchange data during inference (masks are tiled
identically, layers.py:11-13), so the engine shards the *ciphertext batch*
contiguously across ranks (one process per GPU), each rank generating its
evaluation keys from the shared seed (zero key traffic), and the only
collective is the final gather of the decrypted logits -- no data-path
collective, weak scaling.
"""

from __future__ import annotations

import numpy as np

from . import driver, planner


def shard_range(n_items: int, rank: int, world: int):
    """Contiguous [start, stop) slice of n_items for rank (sizes differ by at most one)."""
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def run_sharded(m, samples, params, backend, group=None, fused=True):
    """Encrypted inference of ``samples`` sharded over the ranks of ``group``.

    Every rank calls this with the full sample list; rank r packs and runs the
    ciphertext groups in its shard, then the per-sample logits are gathered so
    every rank returns the full, ordered output list.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    plan = planner.footprint(m, params)
    groups = [samples[i:i + plan.capacity] for i in range(0, len(samples), plan.capacity)]
    lo, hi = shard_range(len(groups), rank, world)
    mine = groups[lo:hi]
    local = []
    if mine:
        planes = driver.pack_groups(m, mine, plan)
        outs, _ = driver.infer_batch(m, planes, params, plan, backend, counts=[len(g) for g in mine], fused=fused)
        local = [np.asarray(y) for grp in outs for y in grp]
    if world == 1:
        return local
    gathered = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    return [y for part in gathered for y in part]
