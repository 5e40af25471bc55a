#!/usr/bin/env python
"""Measurements of the rows either side of the embed path:
one JSON line per row, kernel times with CUDA events on the launching stream,
HBM/PCIe fractions against MEASURED_PEAKS.json, the numpy restatement
(oracle/formats.py) timed on the host as the CPU baseline.

    python tools/bench_rows.py [--rows engine,ingest,layout] [--steps K]

* engine : FrameEngine (device-resident Engine.tick) on C3 data -- online SOM
           tick + model preparation + full re-projection of 2^20 points + the
           FramePoints record written into mapped pinned memory, per frame.
* ingest : a 10M x 32 big-endian FCS image in pinned memory -> zscore'd
           device dataset (H2D, decode, statistics x2, transform).
* layout : one force-layout step at g = 4096 (k_g = 8 graph).
"""

from __future__ import annotations

import argparse
import json
import statistics
import struct
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2201_00701_b200 as esom  # noqa: E402
from paper_2201_00701_b200 import _dev, _lib, datagen  # noqa: E402


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return j.get("hbm_gbs", 6541.8)
    return 6650.0


def timed(fn, reps=5):
    """Median device ms of fn() on the current stream (after one warm call)."""
    fn()
    st = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def fcs_image(points: np.ndarray) -> bytes:
    """Minimal FCS3.0 list-mode writer, big endian (test/bench infrastructure)."""
    n, d = points.shape
    kws = [("$PAR", str(d)), ("$TOT", str(n)), ("$DATATYPE", "F"), ("$BYTEORD", "4,3,2,1"), ("$MODE", "L")]
    kws += [(f"$P{i + 1}B", "32") for i in range(d)] + [(f"$P{i + 1}N", f"ch{i}") for i in range(d)]
    text = b"/" + b"".join(k.encode() + b"/" + v.encode() + b"/" for k, v in kws)
    t0 = 58
    t1 = t0 + len(text) - 1
    d0 = t1 + 1
    d1 = d0 + 4 * n * d - 1
    hdr = b"FCS3.0    " + b"".join(f"{v:>8d}".encode() for v in (t0, t1, d0, d1 if d1 < 10**8 else 0, 0, 0))
    hdr = hdr.ljust(58, b" ")
    return hdr + text + points.astype(">f4").tobytes()


def row_engine(steps):
    pts = datagen.gaussians_f32(16, 1 << 20, 32, seed=1)
    eng = esom.FrameEngine(pts, seed=7, k=16, grid=(16, 16))
    n = pts.shape[0]
    for _ in range(3):
        eng.tick()
        eng.frame_record()
    dev_ms = timed(lambda: eng.tick(), reps=steps)
    wall = []
    for _ in range(steps):
        t0 = time.perf_counter()
        eng.tick()
        rec = eng.frame_record()
        wall.append(time.perf_counter() - t0)
    s = eng.session
    col = s.colors(0)
    buf = s._frame
    from paper_2201_00701_b200.protocol import pack_frame_points

    pack_ms = timed(lambda: pack_frame_points(s.positions, col, 1, buf), reps=steps)
    nbytes = len(rec)
    e2e_s = statistics.median(wall)
    return {"row": "engine", "workload": "FrameEngine on C3 data: 2^20x32, 16x16 SOM, k=16; online SOM tick (256 "
                                         "samples) + full re-projection + FramePoints record into mapped pinned memory",
            "frame_ms_device": dev_ms, "fps_device": 1e3 / dev_ms,
            "e2e": {"fps": 1.0 / e2e_s, "points_per_s": n / e2e_s, "ms": 1e3 * e2e_s, "h2d_bytes_per_step": 256 * 8,
                    "d2h_bytes_per_step": nbytes,
                    "how": "wall clock of tick() + frame_record() (wire bytes readable on the host), median"},
            "pack_kernel": {"ms": pack_ms, "bytes": nbytes, "GBps_over_pcie": nbytes / pack_ms / 1e6,
                            "note": "esom_frame_points_pack writing 13+9n bytes straight into pinned host memory"}}


def row_ingest(steps):
    n, d = 10_000_000, 32
    pts = datagen.gaussians_f32(16, n, d, seed=1) * np.float32(100.0)
    img = fcs_image(pts)
    pinned = torch.empty(len(img), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(img, np.uint8)
    del img
    spec = esom.TransformSpec.uniform("zscore", d)
    esom.apply_transform(esom.parse_fcs(pinned), spec)  # warm
    wall = []
    for _ in range(max(3, steps // 4)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ds = esom.apply_transform(esom.parse_fcs(pinned), spec)
        torch.cuda.synchronize()
        wall.append(time.perf_counter() - t0)
    # kernels alone on resident buffers
    dev = torch.device("cuda")
    raw = torch.empty(4 * n * d, dtype=torch.uint8, device=dev)
    raw.copy_(pinned[pinned.numel() - 4 * n * d:])
    X = torch.empty((n, d), dtype=torch.float32, device=dev)
    flag = _dev.new_flag(dev)
    st = _dev.stream_handle(dev)
    dec_ms = timed(lambda: _lib.call("esom_fcs_decode", _dev.ptr(raw), n * d, 1, _dev.ptr(X), _dev.ptr(flag), st),
                   reps=steps)
    out = torch.empty((4, d), dtype=torch.float64, device=dev)
    ws = torch.empty(_lib.load().esom_dim_stats_workspace_bytes(n, d), dtype=torch.uint8, device=dev)
    stats_ms = timed(lambda: _lib.call("esom_dim_stats", _dev.ptr(X), n, d, _dev.ptr(out[0]), _dev.ptr(out[1]),
                                       _dev.ptr(out[2]), _dev.ptr(out[3]), _dev.ptr(ws), ws.numel(), st), reps=steps)
    kind = torch.full((d,), 2, dtype=torch.int32, device=dev)
    Y = torch.empty_like(X)
    xf_ms = timed(lambda: _lib.call("esom_apply_transform", _dev.ptr(X), n, d, _dev.ptr(kind), 0, 0,
                                    _dev.ptr(out[0]), _dev.ptr(out[1]), _dev.ptr(out[2]), _dev.ptr(out[3]),
                                    _dev.ptr(Y), _dev.ptr(flag), st), reps=steps)
    hbm = peaks()
    vals = n * d

    def kern(ms, bytes_per_value):
        gbs = vals * bytes_per_value / ms / 1e6
        return {"ms": ms, "alg_bytes_per_value": bytes_per_value, "GBps": gbs, "hbm_frac": gbs / hbm}

    # CPU baseline: the reference's numpy path on a bounded sample (1M rows)
    from oracle import formats as F

    m = 1_000_000
    sub = np.frombuffer(pinned.numpy()[pinned.numel() - 4 * n * d:][:4 * m * d].tobytes(), np.uint8)
    t0 = time.perf_counter()
    p = F.fcs_decode(sub, m, d, True)
    stt = F.dim_stats(p)
    z = F.apply_transform(p, ["zscore"] * d, stt)
    F.dim_stats(z)
    cpu_s = time.perf_counter() - t0
    return {"row": "ingest", "workload": "10M x 32 big-endian FCS image in pinned memory -> zscore'd device dataset",
            "e2e": {"points_per_s": n / statistics.median(wall), "ms": 1e3 * statistics.median(wall),
                    "h2d_bytes_per_step": 4 * n * d, "how": "parse_fcs(pinned image) + apply_transform(zscore), wall"},
            "kernels": {"fcs_decode": kern(dec_ms, 8), "dim_stats (2 passes)": kern(stats_ms, 8),
                        "transform": kern(xf_ms, 8)},
            "cpu_baseline": {"points_per_s": m / cpu_s, "cores": 1, "kind": "port",
                             "sample": f"{m} rows: numpy frombuffer/astype + stats + zscore + stats "
                                       "(oracle/formats.py, the reference's numpy ops)"}}


def row_layout(steps):
    g = 4096
    hi = datagen.gaussians(16, g, 32, seed=7)[0].astype(np.float32)
    H = torch.from_numpy(hi).cuda()
    esom.build_knn_graph(H, 8)  # warm (workspace, first launches)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    edges = esom.build_knn_graph(H, 8)
    torch.cuda.synchronize()
    graph_ms = 1e3 * (time.perf_counter() - t0)
    lo = (datagen.extruded_s(g, seed=2)[:, :2] * 10).astype(np.float32)
    st = esom.LayoutState.for_count(g)
    esom.layout_tick(lo, edges, st)
    wall = []
    for _ in range(steps):
        t0 = time.perf_counter()
        esom.layout_tick(lo, edges, st)
        wall.append(time.perf_counter() - t0)
    from oracle import formats as F

    t0 = time.perf_counter()
    F.layout_tick(lo, edges.pairs, edges.rest, st.velocities, st.stiffness, st.repulsion, 1e-3, st.damping, st.dt)
    cpu_ms = 1e3 * (time.perf_counter() - t0)
    return {"row": "layout", "workload": "force-layout step, g=4096 landmarks, k_g=8 graph (f64)",
            "layout_tick_ms_wall": 1e3 * statistics.median(wall), "build_knn_graph_ms_wall": graph_ms,
            "cpu_baseline": {"ms": cpu_ms, "cores": 1, "kind": "port", "sample": "one numpy layout_tick, g=4096"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="engine,ingest,layout")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for r in a.rows.split(","):
        print(json.dumps({"engine": row_engine, "ingest": row_ingest, "layout": row_layout}[r](a.steps)), flush=True)


if __name__ == "__main__":
    main()
