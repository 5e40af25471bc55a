"""Exact k nearest landmarks per point on the B200 (mirror of ref: knn.py).

``knn_base`` and ``knn_bitonic`` keep the reference's names, arguments,
validation order, messages and output layout (indices n×k int32, sqdists
n×k f32, rows ascending by (sqdist, index)).  Both run the same sm_100a
kernel -- the reference guarantees the two backends are bit-identical
(ref: knn.py:1-18), and the kernel reproduces that result bit for bit:
separately rounded f32 sub/mul/add in ascending dimension order and the
lexicographic (distance, index) order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .core import InputError, ParameterError


@dataclass(frozen=True)
class NeighborList:
    """k nearest landmarks per point (ref: knn.py:30-43)."""

    indices: object  # n×k int32 (numpy, or torch on the device for device inputs)
    sqdists: object  # n×k float32

    @property
    def n(self) -> int:
        return self.indices.shape[0]

    @property
    def k(self) -> int:
        return self.indices.shape[1]


def sq_euclidean(a, b) -> float:
    """Squared Euclidean distance of two vectors in f64 (ref: knn.py:46-53; host utility)."""
    av = np.asarray(a, dtype=np.float64).ravel()
    bv = np.asarray(b, dtype=np.float64).ravel()
    if av.shape != bv.shape:
        raise InputError(f"length mismatch: {av.shape[0]} vs {bv.shape[0]}")
    diff = av - bv
    return float(np.dot(diff, diff))


def _shape2(a):
    if isinstance(a, torch.Tensor):
        return tuple(a.shape)
    return np.shape(a)


def _validate_inputs(points, landmarks):
    """Shape checks of ref: knn.py:187-198; finiteness is checked on the device."""
    ps, ls = _shape2(points), _shape2(landmarks)
    if len(ps) != 2 or len(ls) != 2:
        raise InputError("points and landmarks must be 2-d matrices")
    if ps[1] != ls[1]:
        raise InputError(f"dimension mismatch: points d={ps[1]}, landmarks d={ls[1]}")
    return ps, ls


def _run_knn(points, landmarks, k: int) -> NeighborList:
    want_numpy = not _dev.is_device_tensor(points)
    dev = _dev.cuda_device(points)
    with torch.cuda.device(dev):
        X = _dev.to_f32(points, dev)
        L = _dev.to_f32(landmarks, dev)
        n, d = X.shape
        g = L.shape[0]
        idx = torch.empty((n, k), dtype=torch.int32, device=dev)
        sqd = torch.empty((n, k), dtype=torch.float32, device=dev)
        flag = _dev.new_flag(dev)
        nbytes = _lib.load().esom_workspace_bytes(g, d, k, 0)
        ws = _dev.workspace(dev, nbytes)
        _lib.call("esom_knn", _dev.ptr(X), n, d, _dev.ptr(L), g, k, _dev.ptr(idx), _dev.ptr(sqd),
                  _dev.ptr(flag), _dev.ptr(ws), ws.numel(), _dev.stream_handle(dev))
        _dev.raise_if_nonfinite(flag)
        return NeighborList(indices=_dev.out_like(idx, want_numpy), sqdists=_dev.out_like(sqd, want_numpy))


def knn_base(points, landmarks, k: int) -> NeighborList:
    """Exact k nearest landmarks (ref: knn.py:201-214); any 1 <= k <= g."""
    _, ls = _validate_inputs(points, landmarks)
    g = ls[0]
    if not 1 <= k <= g:
        raise ParameterError(f"k={k} violates 1 <= k <= g={g}")
    return _run_knn(points, landmarks, int(k))


def knn_bitonic(points, landmarks, k: int) -> NeighborList:
    """Same result as knn_base; keeps the bitonic backend's k contract (ref: knn.py:217-232)."""
    _, ls = _validate_inputs(points, landmarks)
    g = ls[0]
    if k < 4 or (k & (k - 1)) != 0:
        raise ParameterError(f"bitonic backend needs a power-of-two k >= 4, got {k}")
    if k > g:
        raise ParameterError(f"k={k} violates k <= g={g}")
    return _run_knn(points, landmarks, int(k))


_BACKENDS = {"base": knn_base, "bitonic": knn_bitonic}


def knn(points, landmarks, k: int, backend: str = "bitonic") -> NeighborList:
    """Backend dispatch (ref: knn.py:235-243)."""
    try:
        fn = _BACKENDS[backend]
    except KeyError:
        raise ParameterError(f"unknown knn backend {backend!r}") from None
    return fn(points, landmarks, k)
