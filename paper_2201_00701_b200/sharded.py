"""Online trainer ticks when the points are sharded across ranks.

The online ticks (ref: som.py:44-68, graphmodel.py:87-102) are a strictly
sequential walk over ``batch_size`` sampled points, so they do not shard:
every rank draws the SAME global sample indices from its identically seeded
Rng, copies the sampled rows it owns into a B×d buffer (−0.0 elsewhere, so
the sum is exactly the owner's value), ONE all-reduce(sum) of that buffer
(B·d·4 bytes: 32 KB at C3/C4) gives every rank all B rows, and every rank
runs the identical, deterministic on-chip tick -- the landmarks stay
replicated without a broadcast.  (The batch-SOM step, which does shard, is
batch_som.FrameLoop: one all-reduce of the [S | C] statistics.)
"""

from __future__ import annotations

import numpy as np
import torch

from .batch_som import _allreduce_
from .graphmodel import KmeansConfig
from .som import SomConfig, _online_tick


def gather_sample_rows(X_shard: torch.Tensor, start: int, sample_idx, group=None) -> torch.Tensor:
    """B×d f32 rows of the global ``sample_idx`` from row shards
    [start, start + len(X_shard)) spread over the ranks of ``group``."""
    sidx = torch.as_tensor(np.ascontiguousarray(sample_idx, np.int64), device=X_shard.device)
    rows = torch.full((sidx.numel(), X_shard.shape[1]), -0.0, dtype=torch.float32, device=X_shard.device)
    mine = (sidx >= start) & (sidx < start + X_shard.shape[0])
    rows[mine] = X_shard[sidx[mine] - start].float()
    _allreduce_(rows, group)
    return rows


def som_tick_sharded(X_shard: torch.Tensor, start: int, n_total: int, model, cfg: SomConfig, rng, group=None):
    """``som_tick`` over the union of all ranks' shards; returns device hi
    (identical on every rank)."""
    sample_idx = rng.integers(0, n_total, size=cfg.batch_size)  # the same draw on every rank
    rows = gather_sample_rows(X_shard, start, sample_idx, group)
    return _online_tick("som", rows, model, np.arange(rows.shape[0]), cfg.alpha, cfg.sigma)


def kmeans_tick_sharded(X_shard: torch.Tensor, start: int, n_total: int, model, cfg: KmeansConfig, rng, group=None):
    """``kmeans_tick`` over the union of all ranks' shards (see som_tick_sharded)."""
    sample_idx = rng.integers(0, n_total, size=cfg.batch_size)
    rows = gather_sample_rows(X_shard, start, sample_idx, group)
    return _online_tick("kmeans", rows, model, np.arange(rows.shape[0]), cfg.alpha_km)
