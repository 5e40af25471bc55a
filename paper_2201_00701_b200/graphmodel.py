"""Graph supervision mode on the B200 (mirror of ref: graphmodel.py).

``kmeans_tick`` is on the hot path; the landmark graph and
force layout (§8f row 2) run on the device below; graph edits
(duplicate/remove landmark) stay host bookkeeping in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
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


# ---------------------------------------------------------------------------
# Landmark-side graph ops on the device: the k_g-NN
# graph over the landmarks (the exact k-NN kernel with points = landmarks)
# and the force-layout step (esom_layout_tick).  They only matter once
# g >= 4096; the reference runs them in numpy every tick (layout) or every
# REBUILD_CADENCE ticks (graph).

REPULSION_EPS = 1e-3  # ref: graphmodel.py:22
MIN_LANDMARKS = 3  # ref: graphmodel.py:23
DEFAULT_STIFFNESS = 1.0  # ref: graphmodel.py:25-29
DEFAULT_REPULSION = 0.05
DEFAULT_DAMPING = 0.9
DEFAULT_DT = 0.05
DEFAULT_K_G = 3
REBUILD_CADENCE = 10


@dataclass(frozen=True)
class EdgeSet:
    """Undirected landmark graph: pairs e×2 int32 (i < j), rest lengths e f32 (ref: graphmodel.py:33-45)."""

    pairs: np.ndarray
    rest: np.ndarray

    def __len__(self) -> int:
        return self.pairs.shape[0]

    @classmethod
    def empty(cls) -> "EdgeSet":
        return cls(pairs=np.zeros((0, 2), np.int32), rest=np.zeros(0, np.float32))


@dataclass(frozen=True)
class LayoutState:
    """Velocities (g×2 f64) + force-model parameters (ref: graphmodel.py:60-84)."""

    velocities: np.ndarray
    stiffness: float = DEFAULT_STIFFNESS
    repulsion: float = DEFAULT_REPULSION
    damping: float = DEFAULT_DAMPING
    dt: float = DEFAULT_DT

    def __post_init__(self):
        if not 0.0 < self.damping < 1.0:
            raise ParameterError(f"damping must be in (0, 1), got {self.damping}")
        if not self.dt > 0:
            raise ParameterError(f"dt must be > 0, got {self.dt}")

    @classmethod
    def for_count(cls, g: int, **params) -> "LayoutState":
        return cls(velocities=np.zeros((g, 2), np.float64), **params)


def build_knn_graph(hi, k_g: int, scale: float = 1.0) -> EdgeSet:
    """Symmetrised k_g-NN graph over the landmarks (ref: graphmodel.py:105-135).

    The neighbour lists come from the exact device k-NN (bit-identical to
    knn_base); self matches are skipped wherever they fall, the first k_g
    others per row are kept, and an undirected edge keeps the distance of
    its first occurrence in row-major order -- the reference's dict walk,
    vectorised."""
    from .knn import knn_base

    h = hi if isinstance(hi, torch.Tensor) else np.ascontiguousarray(hi, dtype=np.float32)
    g = h.shape[0]
    if not 1 <= k_g < g:
        raise ParameterError(f"k_g={k_g} violates 1 <= k_g < g={g}")
    nb = knn_base(h, h, k_g + 1)
    idx = np.asarray(nb.indices.cpu() if isinstance(nb.indices, torch.Tensor) else nb.indices)
    sqd = np.asarray(nb.sqdists.cpu() if isinstance(nb.sqdists, torch.Tensor) else nb.sqdists)
    return symmetrize_neighbors(idx, sqd, k_g, scale)


def symmetrize_neighbors(idx: np.ndarray, sqd: np.ndarray, k_g: int, scale: float = 1.0) -> EdgeSet:
    """Edges from (k_g + 1)-NN rows of the landmarks against themselves
    (host bookkeeping of build_knn_graph, ref: graphmodel.py:118-135)."""
    g = idx.shape[0]
    rows = np.repeat(np.arange(g, dtype=np.int64), k_g + 1).reshape(g, k_g + 1)
    other = idx != rows
    keep = other & (np.cumsum(other, axis=1) <= k_g)
    i, j, dist2 = rows[keep], idx[keep].astype(np.int64), sqd[keep]
    key = np.minimum(i, j) * g + np.maximum(i, j)
    if key.size == 0:
        return EdgeSet.empty()
    uniq, first = np.unique(key, return_index=True)  # sorted keys, first occurrence in walk order
    pairs = np.stack([uniq // g, uniq % g], axis=1).astype(np.int32)
    rest = (scale * np.sqrt(dist2[first]).astype(np.float64)).astype(np.float32)
    return EdgeSet(pairs=pairs, rest=rest)


def graph_scale_for_unit_rest(hi, k_g: int) -> float:
    """ref: graphmodel.py:138-142"""
    raw = build_knn_graph(hi, k_g, scale=1.0)
    mean = float(raw.rest.mean()) if len(raw) else 0.0
    return 1.0 / mean if mean > 0 else 1.0


def _edge_csr(pairs: np.ndarray, g: int):
    """node -> signed edge ids: first-endpoint edges (e) then second-endpoint
    edges (-e-1), each in edge order (np.add.at's accumulation order)."""
    e = np.arange(pairs.shape[0], dtype=np.int64)
    node = np.concatenate([pairs[:, 0], pairs[:, 1]]).astype(np.int64)
    sid = np.concatenate([e, -e - 1])
    rank = np.concatenate([e, e + pairs.shape[0]])
    order = np.lexsort((rank, node))
    ptr = np.zeros(g + 1, np.int64)
    ptr[1:] = np.bincount(node, minlength=g)[:g]  # (np.add.at here cost ~4 ms at g = 4096)
    return np.cumsum(ptr).astype(np.int32), sid[order].astype(np.int32)


_EDGE_CACHE: dict = {}


def _edge_device(edges, g: int, dev):
    """Device copies of an edge set (pairs, rest, CSR), cached while the same
    EdgeSet arrays are passed again -- the engine rebuilds its graph every
    REBUILD_CADENCE ticks but lays out every tick."""
    key = (dev.index if isinstance(dev, torch.device) else int(dev), g)
    hit = _EDGE_CACHE.get(key)
    if hit is not None and hit[0] is edges.pairs and hit[1] is edges.rest:
        return hit[2]
    pairs = np.ascontiguousarray(edges.pairs, dtype=np.int32).reshape(-1, 2)
    if pairs.size and (int(pairs.min()) < 0 or int(pairs.max()) >= g):
        # the reference's np.add.at raises here (ref: graphmodel.py:160-163); the
        # kernel would read out of bounds
        bad = int(pairs.max()) if int(pairs.max()) >= g else int(pairs.min())
        raise IndexError(f"index {bad} is out of bounds for axis 0 with size {g}")
    ptr, sid = _edge_csr(pairs, g)
    out = (torch.from_numpy(pairs.copy()).to(dev),
           torch.from_numpy(np.ascontiguousarray(edges.rest, dtype=np.float32)).to(dev),
           torch.from_numpy(ptr).to(dev), torch.from_numpy(sid).to(dev))
    _EDGE_CACHE.clear()
    _EDGE_CACHE[key] = (edges.pairs, edges.rest, out)  # holds the arrays: identity stays valid
    return out


def _layout_dev(lo, edges: EdgeSet, st: LayoutState, pinned_rows, want_forces: bool):
    lo_np = np.ascontiguousarray(np.asarray(lo.cpu() if isinstance(lo, torch.Tensor) else lo), dtype=np.float32)
    g = lo_np.shape[0]
    vel = np.asarray(st.velocities, dtype=np.float64)
    if vel.shape != lo_np.shape:
        raise ParameterError("velocity matrix shape does not match layout")
    dev = _dev.cuda_device(lo)
    pin = np.zeros(g, np.uint8)
    for r in pinned_rows:
        pin[int(r)] = 1
    with torch.cuda.device(dev):
        P, R, CP, CE = _edge_device(edges, g, dev)
        L = torch.from_numpy(lo_np).to(dev)
        PN = torch.from_numpy(pin).to(dev)
        V = torch.from_numpy(vel.copy()).to(dev)
        out = torch.empty_like(L)
        Fo = torch.empty((g, 2), dtype=torch.float64, device=dev) if want_forces else None
        _lib.call("esom_layout_tick", _dev.ptr(L), g, _dev.ptr(P), _dev.ptr(R), _dev.ptr(CP), _dev.ptr(CE),
                  _dev.ptr(PN), float(st.stiffness), float(st.repulsion), REPULSION_EPS, float(st.damping),
                  float(st.dt), _dev.ptr(V), _dev.ptr(out), _dev.ptr(Fo), _dev.stream_handle(dev))
        return out.cpu().numpy(), V.cpu().numpy(), (Fo.cpu().numpy() if want_forces else None)


def net_forces(lo, edges: EdgeSet, st: LayoutState) -> np.ndarray:
    """Spring + repulsion forces g×2 f64 (ref: graphmodel.py:145-167), on the device."""
    return _layout_dev(lo, edges, st, (), True)[2]


def layout_tick(lo, edges: EdgeSet, st: LayoutState, pinned_rows=()):
    """One semi-implicit Euler step -> (new lo f32, new velocities f64) (ref: graphmodel.py:170-192)."""
    new_lo, vel, _ = _layout_dev(lo, edges, st, pinned_rows, False)
    return new_lo, vel
