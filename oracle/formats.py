"""numpy restatements of the data formats either side of the embed path
(SURVEY.md §8f rows 1-4): frame colours, the FramePoints wire record, the
FCS DATA decode, per-dimension statistics, dataset transforms and the
landmark-side graph ops.

TEST INFRASTRUCTURE ONLY (like oracle.py): imported by tests/ and bench.py's
CPU-baseline / ``--impl reference`` leg, never by the product package.  Each
function cites the reference lines it restates; tests/golden/make_golden_frames.py
pins them against the reference run in the build container.
"""

from __future__ import annotations

import struct

import numpy as np

TAG_FRAME_POINTS = 0x31  # ref: protocol.py:33


def color_channel(points, col_min, col_max, color_dim: int) -> np.ndarray:
    """ref: engine.py:144-153 (f64 min-max quantisation, rint, u8)."""
    vals = np.asarray(points)[:, color_dim].astype(np.float64)
    lo = float(col_min[color_dim])
    span = float(col_max[color_dim]) - lo
    if span <= 0:
        return np.full(vals.shape[0], 128, np.uint8)
    return np.rint((vals - lo) / span * 255.0).astype(np.uint8)


def frame_points_record(frame_id: int, positions, colors) -> bytes:
    """protocol.encode(FramePoints(...)) (ref: protocol.py:205-210, 216-218)."""
    pos = np.ascontiguousarray(positions, dtype="<f4")
    col = np.ascontiguousarray(colors, dtype=np.uint8)
    body = struct.pack("<II", frame_id, pos.shape[0]) + pos.tobytes() + col.tobytes()
    return struct.pack("<I", 1 + len(body)) + bytes([TAG_FRAME_POINTS]) + body


def fcs_decode(data_bytes, n: int, d: int, big_endian: bool) -> np.ndarray:
    """ref: io.py:124-125 (np.frombuffer in $BYTEORD order, astype('<f4'))."""
    dt = np.dtype(">f4" if big_endian else "<f4")
    return np.frombuffer(data_bytes, dtype=dt, count=n * d).astype("<f4").reshape(n, d)


def dim_stats(points):
    """ref: core.py:54-69 -> (min, max, mean, sd) f64 arrays."""
    m = np.asarray(points).astype(np.float64)
    return m.min(axis=0), m.max(axis=0), m.mean(axis=0), m.std(axis=0)


def apply_transform(points, entries, stats=None) -> np.ndarray:
    """ref: io.py:205-229 (f64 per column, cast to f32)."""
    cols = np.asarray(points).astype(np.float64)
    mn, mx, mean, sd = stats if stats is not None else dim_stats(points)
    out = np.empty_like(cols)
    for c, e in enumerate(entries):
        x = cols[:, c]
        if e == "none":
            out[:, c] = x
        elif e == "minmax":
            span = mx[c] - mn[c]
            out[:, c] = 0.5 if span <= 0 else (x - mn[c]) / span
        elif e == "zscore":
            out[:, c] = 0.0 if sd[c] <= 0 else (x - mean[c]) / sd[c]
        else:
            out[:, c] = e[1] * x + e[2]
    return out.astype(np.float32)


def net_forces(lo, pairs, rest, stiffness: float, repulsion: float, eps: float) -> np.ndarray:
    """ref: graphmodel.py:138-167 (springs on the edges + all-pairs repulsion), f64."""
    pos = np.asarray(lo, dtype=np.float64)
    g = pos.shape[0]
    f = np.zeros((g, 2), np.float64)
    for (i, j), r in zip(np.asarray(pairs), np.asarray(rest)):
        dx = pos[j] - pos[i]
        dist = np.sqrt(dx @ dx)
        if dist > 0:
            pull = stiffness * (dist - r) / dist * dx
            f[i] += pull
            f[j] -= pull
    diff = pos[:, None, :] - pos[None, :, :]
    r2 = (diff * diff).sum(axis=2)
    inv = repulsion / np.power(r2 + eps, 1.5)
    np.fill_diagonal(inv, 0.0)
    f += (inv[:, :, None] * diff).sum(axis=1)
    return f


def layout_tick(lo, pairs, rest, velocities, stiffness, repulsion, eps, damping, dt, pinned_rows=()):
    """ref: graphmodel.py:170-192 (semi-implicit Euler, pinned rows frozen)."""
    pos = np.asarray(lo, dtype=np.float64)
    vel = damping * (np.asarray(velocities, np.float64) + dt * net_forces(pos, pairs, rest, stiffness, repulsion,
                                                                          eps))
    new_lo = (pos + dt * vel).astype(np.float32)
    pin = np.asarray(list(pinned_rows), dtype=np.int64)
    if pin.size:
        vel[pin] = 0.0
        new_lo[pin] = np.asarray(lo, np.float32)[pin]
    return new_lo, vel


def fit_hi_for_new_landmark(pos2d, hi, lo, eps: float = 1e-6) -> np.ndarray:
    """ref: som.py:82-101 (inverse-distance weighting in f64; exact hit -> copy)."""
    pos = np.asarray(pos2d, dtype=np.float64).ravel()
    diff = np.asarray(lo, np.float64) - pos[None, :]
    d2 = (diff * diff).sum(axis=1)
    j = int(np.argmin(d2))
    if d2[j] < eps:
        return np.asarray(hi, np.float32)[j].copy()
    w = 1.0 / (d2 + eps)
    return ((w @ np.asarray(hi, np.float64)) / w.sum()).astype(np.float32)
