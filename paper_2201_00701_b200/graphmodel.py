"""Online k-means landmark training on the B200 (mirror of ref: graphmodel.py:48-102).

Only ``kmeans_tick`` is on the hot path; the force layout
and graph edits are g-sized host work and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import ParameterError, points_of
from .som import _online_tick


@dataclass(frozen=True)
class KmeansConfig:
    """ref: graphmodel.py:48-57"""

    alpha_km: float = 0.05
    batch_size: int = 256

    def __post_init__(self):
        if not 0.0 < self.alpha_km <= 1.0:
            raise ParameterError(f"alpha_km must be in (0, 1], got {self.alpha_km}")
        if self.batch_size < 1:
            raise ParameterError(f"batch_size must be >= 1, got {self.batch_size}")


def kmeans_tick(dataset, model, cfg: KmeansConfig, rng):
    """One online k-means tick: each drawn sample moves only its BMU (ref: graphmodel.py:87-102)."""
    n = points_of(dataset).shape[0]
    sample_idx = rng.integers(0, n, size=cfg.batch_size)
    return _online_tick("kmeans", dataset, model, sample_idx, cfg.alpha_km)
