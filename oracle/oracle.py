"""ctypes front end of the CPU checker (oracle/esom_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / ``--impl reference`` leg -- never by the product
package.  Every function restates the reference function it names (see the
file:line citations in esom_oracle.c) and is pinned against fixtures made by
running the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def build() -> Path:
    """Compile the checker with its Makefile (gcc; no reference sources)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build()
    L = C.CDLL(str(_LIB_PATH))
    L.oracle_knn_base.argtypes = [_f32p, C.c_int64, C.c_int, _f32p, C.c_int, C.c_int, _i32p, _f32p]
    L.oracle_knn_bitonic.argtypes = L.oracle_knn_base.argtypes
    L.oracle_scores.argtypes = [_f32p, C.c_int64, C.c_int, _f64p]
    L.oracle_project.argtypes = [_f32p, C.c_int64, C.c_int, _f32p, _f32p, _i32p, _f64p, C.c_int, _f32p]
    L.oracle_embed.argtypes = [_f32p, C.c_int64, C.c_int, _f32p, _f32p, C.c_int, C.c_int, C.c_int, _f32p]
    L.oracle_embed_mt.argtypes = L.oracle_embed.argtypes + [C.c_int]
    L.oracle_som_tick.argtypes = [_f32p, C.c_int, _i64p, C.c_int, _f32p, _f32p, C.c_int, C.c_double, C.c_double]
    L.oracle_kmeans_tick.argtypes = [_f32p, C.c_int, _i64p, C.c_int, _f32p, C.c_int, C.c_double]
    L.oracle_batch_som_accumulate.argtypes = [_f32p, C.c_int64, C.c_int, _f32p, C.c_int, _f64p, _i64p]
    L.oracle_batch_som_update.argtypes = [_f64p, _i64p, _f32p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _f32p]
    L.oracle_quantization_error.argtypes = [_f32p, C.c_int64, C.c_int, _f32p, C.c_int]
    L.oracle_quantization_error.restype = C.c_double
    for f in (L.oracle_knn_base, L.oracle_knn_bitonic, L.oracle_scores, L.oracle_project,
              L.oracle_embed, L.oracle_embed_mt, L.oracle_som_tick, L.oracle_kmeans_tick,
              L.oracle_batch_som_accumulate, L.oracle_batch_som_update):
        f.restype = None
    _lib = L
    return L


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def knn(points, landmarks, k: int, backend: str = "base"):
    """(indices n×k int32, sqdists n×k f32) -- ref: knn.py:201-232."""
    p, lm = _f32(points), _f32(landmarks)
    n, d = p.shape
    g = lm.shape[0]
    idx = np.empty((n, k), np.int32)
    sqd = np.empty((n, k), np.float32)
    fn = lib().oracle_knn_bitonic if backend == "bitonic" else lib().oracle_knn_base
    fn(p, n, d, lm, g, k, idx, sqd)
    return idx, sqd


def scores(sqdists):
    """n×k f64 scores -- ref: projection.py:38-65."""
    s = _f32(np.atleast_2d(sqdists))
    out = np.empty(s.shape, np.float64)
    lib().oracle_scores(s, s.shape[0], s.shape[1], out)
    return out


def project(points, hi, lo, indices, score_rows):
    """n×2 f32 -- ref: projection.py:68-121 (mixed-precision contract)."""
    p = _f32(points)
    idx = np.ascontiguousarray(indices, np.int32)
    sc = np.ascontiguousarray(score_rows, np.float64)
    out = np.empty((p.shape[0], 2), np.float32)
    lib().oracle_project(p, p.shape[0], p.shape[1], _f32(hi), _f32(lo), idx, sc, idx.shape[1], out)
    return out


def embed(points, hi, lo, k: int, backend: str = "base", threads: int = 1):
    """n×2 f32 -- ref: projection.py:220-245 (row-sharded over threads)."""
    p = _f32(points)
    h = _f32(hi)
    out = np.empty((p.shape[0], 2), np.float32)
    b = 1 if backend == "bitonic" else 0
    if threads > 1:
        lib().oracle_embed_mt(p, p.shape[0], p.shape[1], h, _f32(lo), h.shape[0], k, b, out, threads)
    else:
        lib().oracle_embed(p, p.shape[0], p.shape[1], h, _f32(lo), h.shape[0], k, b, out)
    return out


def som_tick(points, hi, lo, sample_idx, sigma: float, alpha: float):
    """g×d f32 -- ref: som.py:44-68, with the host-drawn sample indices."""
    p = _f32(points)
    h = _f32(hi).copy()
    s = np.ascontiguousarray(sample_idx, np.int64)
    lib().oracle_som_tick(p, p.shape[1], s, s.shape[0], h, _f32(lo), h.shape[0], sigma, alpha)
    return h


def kmeans_tick(points, hi, sample_idx, alpha_km: float):
    """g×d f32 -- ref: graphmodel.py:87-102."""
    p = _f32(points)
    h = _f32(hi).copy()
    s = np.ascontiguousarray(sample_idx, np.int64)
    lib().oracle_kmeans_tick(p, p.shape[1], s, s.shape[0], h, h.shape[0], alpha_km)
    return h


def batch_som_accumulate(points, hi):
    p, h = _f32(points), _f32(hi)
    g, d = h.shape
    S = np.empty((g, d), np.float64)
    Cn = np.empty(g, np.int64)
    lib().oracle_batch_som_accumulate(p, p.shape[0], d, h, g, S, Cn)
    return S, Cn


def batch_som_update(S, Cn, lo, hi, sigma: float, alpha: float, mode: int = 0):
    h = _f32(hi).copy()
    g, d = h.shape
    lib().oracle_batch_som_update(np.ascontiguousarray(S, np.float64),
                                  np.ascontiguousarray(Cn, np.int64), _f32(lo), g, d,
                                  sigma, alpha, mode, h)
    return h


def batch_som_step(points, hi, lo, sigma: float, alpha: float, mode: int = 0):
    S, Cn = batch_som_accumulate(points, hi)
    return batch_som_update(S, Cn, lo, hi, sigma, alpha, mode)


def batch_som_accumulate_fx(points, hi, fx: int):
    """The device's exact statistics (batch_som.py): BMU = exact f32 nearest
    landmark (knn_base k = 1), S_b = sum of round(x 2^fx) as int64, C_b = count.
    Integer sums: any split of the points gives the same S, C."""
    p = _f32(points)
    g, d = _f32(hi).shape
    b = knn(p, hi, 1)[0][:, 0].astype(np.int64)
    q = np.rint(p.astype(np.float64) * np.ldexp(1.0, fx)).astype(np.int64)  # round half even, like __double2ll_rn
    S = np.zeros((g, d), np.int64)
    np.add.at(S, b, q)
    return S, np.bincount(b, minlength=g).astype(np.int64)


def batch_som_update_fx(S_int, Cn, fx: int, lo, hi, sigma: float, alpha: float, mode: int = 0):
    """batch_som_update on the fixed-point statistics (S = S_int 2^-fx, exact in f64 below 2^53)."""
    return batch_som_update(np.asarray(S_int, np.int64).astype(np.float64) * np.ldexp(1.0, -fx), Cn, lo, hi,
                            sigma, alpha, mode)


def quantization_error(points, hi) -> float:
    p, h = _f32(points), _f32(hi)
    return float(lib().oracle_quantization_error(p, p.shape[0], p.shape[1], h, h.shape[0]))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1
