"""Minibatch sharding across GPUs.

Minibatches are independent under per-root streams (each root's stream seed
is keyed by its global (batch, position), cli.cpp:401-408 /
trainer.cpp:200-206), so a step's k batches split into contiguous ranges per
rank with no collective on the data path; the union of the per-rank results
equals the single-device result batch for batch.
"""
from __future__ import annotations

import numpy as np


def batch_range(k: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous batch range of `rank` (same split rule as the reference's
    worker_component_range, trainer.cpp:214-219)."""
    return k * rank // world, k * (rank + 1) // world


def shard(roots: np.ndarray, batch_off: np.ndarray, seeds: np.ndarray, rank: int, world: int):
    """The rank's slice of a flat (roots, batch_off, seeds) call."""
    k = len(batch_off) - 1
    b0, b1 = batch_range(k, rank, world)
    r0, r1 = int(batch_off[b0]), int(batch_off[b1])
    return roots[r0:r1], batch_off[b0:b1 + 1] - r0, seeds[r0:r1]


def worker_component_range(n_components: int, rank: int, world: int) -> tuple[int, int]:
    """The contiguous component range rank r of world owns within one batch
    (trainer.cpp:214-219), the slice the reference's DDP worker trains on
    (slice_components, trainer.cpp:342-343)."""
    return n_components * rank // world, n_components * (rank + 1) // world
