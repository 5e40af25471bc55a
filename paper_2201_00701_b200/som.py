"""SOM landmark training on the B200 (mirror of ref: som.py).

``som_tick`` keeps the reference semantics exactly: ``batch_size`` sample
indices are drawn on the host from the caller's Rng (ref: som.py:57) and
applied *sequentially* in f64 by one CTA (BMU = first index of the f64
minimum, then hi += (alpha*h_j)(x - hi) with h over layout distances).
``quantization_error`` reduces the exact nearest-landmark squared distances
on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .core import InputError, ParameterError, points_of

FIT_EPS = 1e-6  # ref: som.py:17


@dataclass(frozen=True)
class SomConfig:
    """ref: som.py:20-32"""

    sigma: float = 1.0
    alpha: float = 0.1
    batch_size: int = 256

    def __post_init__(self):
        if not self.sigma > 0:
            raise ParameterError(f"sigma must be > 0, got {self.sigma}")
        if not 0.0 <= self.alpha <= 1.0:
            raise ParameterError(f"alpha must be in [0, 1], got {self.alpha}")
        if self.batch_size < 1:
            raise ParameterError(f"batch_size must be >= 1, got {self.batch_size}")


def bmu(point, hi) -> int:
    """Index of the nearest landmark in f64, ties to the lower index (ref: som.py:35-41).

    Single-vector host utility, identical to the reference; the batched,
    accelerated BMU lives in the device trainers and ``knn``.
    """
    p = np.asarray(point, dtype=np.float64).ravel()
    h = np.asarray(hi, dtype=np.float64)
    diff = h - p[None, :]
    return int(np.argmin(np.einsum("gd,gd->g", diff, diff)))


def _online_tick(kind: str, dataset, model, sample_idx, a: float, sigma: float = 1.0):
    pts = points_of(dataset)
    want_numpy = not _dev.is_device_tensor(pts)
    dev = _dev.cuda_device(pts)
    with torch.cuda.device(dev):
        hi = _dev.to_f32(model.hi, dev).clone()
        g, d = hi.shape
        if pts.shape[1] != d:
            raise InputError(f"points have d={pts.shape[1]}, model has d={d}")
        if want_numpy and not isinstance(sample_idx, torch.Tensor):
            # host dataset: the tick reads only the sampled rows, so gather them on the
            # host and upload B×d (not the whole n×d matrix every tick); same sample
            # order, so the sequential update is unchanged
            rows = np.asarray(pts, dtype=np.float32)[np.asarray(sample_idx, np.int64)]
            X = _dev.to_dev_async(np.ascontiguousarray(rows), dev)
            sidx = _dev.to_dev_async(np.arange(rows.shape[0], dtype=np.int64), dev)
        else:
            X = _dev.to_f32(pts, dev)
            sidx = _dev.to_dev_async(np.asarray(sample_idx, np.int64), dev) if not isinstance(
                sample_idx, torch.Tensor) else sample_idx.to(device=dev, dtype=torch.int64).contiguous()
        nb = _lib.load().esom_tick_workspace_bytes(g, d)
        ws = _dev.workspace(dev, nb, slot="tick")
        st = _dev.stream_handle(dev)
        if kind == "som":
            lo = (_dev.to_f32(model.lo, dev) if isinstance(model.lo, torch.Tensor)
                  else _dev.to_dev_async(np.asarray(model.lo, np.float32), dev))
            _lib.call("esom_som_tick", _dev.ptr(X), d, _dev.ptr(sidx), sidx.numel(), _dev.ptr(hi), _dev.ptr(lo), g,
                      float(sigma), float(a), _dev.ptr(ws), ws.numel(), st)
        else:
            _lib.call("esom_kmeans_tick", _dev.ptr(X), d, _dev.ptr(sidx), sidx.numel(), _dev.ptr(hi), g, float(a),
                      _dev.ptr(ws), ws.numel(), st)
        return _dev.out_like(hi, want_numpy)


def som_tick(dataset, model, cfg: SomConfig, rng):
    """One online SOM tick; returns the updated hi (ref: som.py:44-68)."""
    n = points_of(dataset).shape[0]
    sample_idx = rng.integers(0, n, size=cfg.batch_size)  # host draw, same stream as the reference
    return _online_tick("som", dataset, model, sample_idx, cfg.alpha, cfg.sigma)


def quantization_error(dataset, hi) -> float:
    """Mean nearest-landmark squared distance (ref: som.py:71-79), reduced on the device."""
    pts = points_of(dataset)
    dev = _dev.cuda_device(pts)
    with torch.cuda.device(dev):
        X = _dev.to_f32(pts, dev)
        H = _dev.to_f32(hi, dev)
        n, d = X.shape
        g = H.shape[0]
        qe = torch.zeros(1, dtype=torch.float64, device=dev)
        flag = _dev.new_flag(dev)
        ws = _dev.workspace(dev, _lib.load().esom_workspace_bytes(g, d, 1, 0))
        _lib.call("esom_bmu_accumulate", _dev.ptr(X), n, d, _dev.ptr(H), g, _dev.ptr(ws), ws.numel(), 0, 0, 0, 0,
                  _dev.ptr(qe), _dev.ptr(flag), _dev.stream_handle(dev))
        _dev.raise_if_nonfinite(flag)
        return float(qe.item()) / max(n, 1)


def fit_hi_for_new_landmark(pos2d, model) -> np.ndarray:
    """hi row for a landmark added at a layout position: inverse-distance
    weighting over the layout, an exact hit copies that landmark's hi
    (ref: som.py:82-101), computed by one CTA (esom_fit_hi)."""
    if model.hi.shape[0] == 0:
        raise InputError("empty model")
    pos = np.asarray(pos2d, dtype=np.float64).ravel()
    if pos.shape[0] != 2:
        raise InputError("pos2d must be a 2-vector")
    dev = _dev.cuda_device(model.hi)
    with torch.cuda.device(dev):
        hi = _dev.to_f32(model.hi, dev)
        lo = _dev.to_f32(model.lo, dev)
        g, d = hi.shape
        out = torch.empty(d, dtype=torch.float32, device=dev)
        _lib.call("esom_fit_hi", _dev.ptr(hi), _dev.ptr(lo), g, d, float(pos[0]), float(pos[1]), FIT_EPS,
                  _dev.ptr(out), _dev.stream_handle(dev))
        return out.cpu().numpy()
