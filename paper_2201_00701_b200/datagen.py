"""Synthetic inputs with the reference's generators (ref: datagen.py:9-28),
so CPU and GPU arms (and the golden fixtures) see bit-identical data."""

from __future__ import annotations

import numpy as np

from .core import ParameterError, Rng


def uniform(n: int, d: int, seed: int) -> np.ndarray:
    """n×d points uniform in [0, 1) (ref: datagen.py:9-13)."""
    if n < 1 or d < 1:
        raise ParameterError("need n >= 1 and d >= 1")
    return Rng(seed).uniform(0.0, 1.0, size=(n, d)).astype(np.float32)


def gaussians(c: int, n: int, d: int, seed: int, sd: float = 0.5, center_span: float = 10.0):
    """c spherical clusters: (points f32, labels int64) (ref: datagen.py:16-28)."""
    if c < 1:
        raise ParameterError("need at least one cluster")
    rng = Rng(seed)
    centers = rng.uniform(0.0, center_span, size=(c, d))
    labels = rng.integers(0, c, size=n)
    noise = rng.normal(0.0, 1.0, size=(n, d)) * sd
    return (centers[labels] + noise).astype(np.float32), labels.astype(np.int64)


def extruded_s(n: int, seed: int, noise: float = 0.05) -> np.ndarray:
    """3-D S-curve swept along y (ref: datagen.py:31-44), used by the SOM
    efficacy checks (tests:test_som.py:440-450)."""
    rng = Rng(seed)
    t = rng.uniform(-1.5 * np.pi, 1.5 * np.pi, size=n)
    y = rng.uniform(0.0, 2.0, size=n)
    pts = np.stack([np.sin(t), y, np.sign(t) * (np.cos(t) - 1.0)], axis=1)
    if noise > 0:
        pts = pts + rng.normal(0.0, noise, size=(n, 3))
    return pts.astype(np.float32)


def lattice(rows: int, cols: int) -> np.ndarray:
    """g×2 unit lattice layout, x fastest (ref: engine.py:215-217)."""
    ys, xs = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    return np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.float32)


def som_model(points: np.ndarray, rows: int, cols: int, seed: int):
    """Engine-style initial model: lattice lo, hi = distinct data rows drawn
    by Rng(seed).choice_distinct (ref: engine.py:208-227).  Returns (hi, lo)."""
    g = rows * cols
    idx = Rng(seed).choice_distinct(points.shape[0], g)
    return np.ascontiguousarray(points[idx], np.float32), lattice(rows, cols)


def gaussians_chunks(c: int, n: int, d: int, seed: int, chunk: int = 1 << 18, sd: float = 0.5,
                     center_span: float = 10.0):
    """Yield (start, rows f32) blocks identical to ``gaussians(...)[0][start:start+len]``.

    The reference draws centers, then all labels, then the n×d noise from one
    Philox stream; Generator draws continue the stream across calls, so the
    noise can be produced block by block without holding n×d f64 in memory.
    """
    rng = Rng(seed)
    centers = rng.uniform(0.0, center_span, size=(c, d))
    labels = rng.integers(0, c, size=n)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        noise = rng.normal(0.0, 1.0, size=(m, d)) * sd
        yield s, (centers[labels[s:s + m]] + noise).astype(np.float32)


def gaussians_f32(c: int, n: int, d: int, seed: int, chunk: int = 1 << 18) -> np.ndarray:
    """gaussians(...)[0] assembled block-wise (peak memory ~ n×d×4 bytes)."""
    out = np.empty((n, d), np.float32)
    for s, blk in gaussians_chunks(c, n, d, seed, chunk):
        out[s:s + blk.shape[0]] = blk
    return out


def gaussians_slice(c: int, n: int, d: int, seed: int, start: int, stop: int, pick=None,
                    chunk: int = 1 << 18, sd: float = 0.5, center_span: float = 10.0):
    """Rows [start, stop) of ``gaussians(c, n, d, seed)[0]`` plus the rows at
    indices ``pick`` (any positions in [0, n)), without materialising the
    other rows: the Philox stream is consumed block by block up to
    max(stop, max(pick)) and only the wanted rows are kept.  One rank's
    contiguous shard of the SURVEY §8d dataset, and the landmark rows every
    rank must agree on."""
    pick = np.asarray([] if pick is None else pick, np.int64)
    out = np.empty((stop - start, d), np.float32)
    picked = np.empty((pick.shape[0], d), np.float32)
    end = max(stop, int(pick.max()) + 1 if pick.size else 0)
    rng = Rng(seed)
    centers = rng.uniform(0.0, center_span, size=(c, d))
    labels = rng.integers(0, c, size=n)
    for s in range(0, end, chunk):
        m = min(chunk, n - s)
        noise = rng.normal(0.0, 1.0, size=(m, d)) * sd
        blk = (centers[labels[s:s + m]] + noise).astype(np.float32)
        lo_, hi_ = max(s, start), min(s + m, stop)
        if lo_ < hi_:
            out[lo_ - start:hi_ - start] = blk[lo_ - s:hi_ - s]
        sel = np.nonzero((pick >= s) & (pick < s + m))[0]
        if sel.size:
            picked[sel] = blk[pick[sel] - s]
    return out, picked


def som_model_rows(n: int, rows: int, cols: int, seed: int) -> np.ndarray:
    """The dataset row indices ``som_model`` draws for hi (Rng(seed).choice_distinct)."""
    return Rng(seed).choice_distinct(n, rows * cols)
