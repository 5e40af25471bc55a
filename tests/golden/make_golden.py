"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``embedview`` from /root/reference/pkg/src read-only, builds the
inputs with the reference's own generators and seeds (tests:conftest.py,
tests:test_acceptance.py), and writes

* ``golden.npz``  -- small arrays (inputs are regenerated from seeds; each
  case stores a sha256 of its inputs so a generator drift is caught), and
* ``digests.json`` -- sha256 of reference outputs for cases too large to
  store (the full c01 grid at n = 10^4, C1 and C2/C4/C5-shaped samples).

Nothing at test or bench time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(REF))

from embedview import datagen as rdg  # noqa: E402
from embedview.core import Dataset, LandmarkModel, Rng  # noqa: E402
from embedview.graphmodel import KmeansConfig, kmeans_tick  # noqa: E402
from embedview.knn import knn_base, knn_bitonic  # noqa: E402
from embedview.projection import _scores_matrix, embed, project_neighbors, project_point, scores  # noqa: E402
from embedview.core import EmbedParams  # noqa: E402
from embedview.som import SomConfig, quantization_error, som_tick  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def lattice(rows, cols):
    ys, xs = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    return np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.float32)


def som_model(points, rows, cols, seed):
    idx = Rng(seed).choice_distinct(points.shape[0], rows * cols)
    return np.ascontiguousarray(points[idx], np.float32), lattice(rows, cols)


def main():
    arrays: dict[str, np.ndarray] = {}
    digests: dict[str, dict] = {}
    t0 = time.time()

    # --- C1: gaussians(8, 10_000, 4, seed=1), 8x8 SOM model, k=8 (BASELINE configs[0]) ---
    pts, _ = rdg.gaussians(8, 10_000, 4, seed=1)
    hi, lo = som_model(pts, 8, 8, seed=2)
    model = LandmarkModel.create(hi, lo)
    nb = knn_base(pts, hi, 8)
    nb2 = knn_bitonic(pts, hi, 8)
    assert np.array_equal(nb.indices, nb2.indices) and np.array_equal(nb.sqdists, nb2.sqdists)
    sc = _scores_matrix(nb.sqdists)
    xy = embed(pts, model, EmbedParams(k=8))
    xyb = embed(pts, model, EmbedParams(k=8), backend="base")
    assert np.array_equal(xy, xyb)
    arrays["c1_idx"] = nb.indices
    arrays["c1_sqd"] = nb.sqdists
    arrays["c1_scores"] = sc
    arrays["c1_xy"] = xy
    digests["c1"] = {"inputs": sha(pts, hi, lo), "idx": sha(nb.indices), "sqd": sha(nb.sqdists),
                     "scores": sha(sc), "xy": sha(xy), "qe": quantization_error(Dataset.from_points(pts), hi)}
    print("c1", time.time() - t0, flush=True)

    # --- c01 grid (tests:test_acceptance.py:37-67): digests of knn_base at n=10^4 ---
    grid = {}
    for seed in (101, 202, 303):
        for d in (2, 16, 64):
            points = rdg.uniform(10_000, d, seed)
            for g in (16, 64, 257, 1024):
                landmarks = rdg.uniform(g, d, seed + g)
                for k in (4, 8, 16, 32, 64):
                    if k > g:
                        continue
                    a = knn_base(points, landmarks, k)
                    grid[f"{seed}_{d}_{g}_{k}"] = {"inputs": sha(points, landmarks),
                                                   "idx": sha(a.indices), "sqd": sha(a.sqdists)}
        print("grid seed", seed, time.time() - t0, flush=True)
    digests["c01_grid"] = grid

    # --- reference test_knn fixtures with random inputs (default_rng based) ---
    gen = np.random.default_rng(20240817)
    p = gen.normal(size=(1000, 8)).astype(np.float32)
    l = gen.normal(size=(257, 8)).astype(np.float32)
    a = knn_base(p, l, 16)
    arrays["sentinel257_points"], arrays["sentinel257_landmarks"] = p, l
    arrays["sentinel257_idx"], arrays["sentinel257_sqd"] = a.indices, a.sqdists

    # --- scores rows (projection.py:38-65) ---
    gen = np.random.default_rng(5)
    rows = [np.array([0.0, 1.0, 4.0], np.float32), np.full(5, 2.0, np.float32), np.zeros(4, np.float32)]
    for k in (3, 4, 8, 16, 32, 64):
        for _ in range(8):
            rows.append(np.sort(gen.random(k) * gen.uniform(1e-3, 1e3)).astype(np.float32))
    for i, r in enumerate(rows):
        arrays[f"scores_in_{i}"] = r
        arrays[f"scores_out_{i}"] = scores(r).scores
    arrays["scores_count"] = np.array([len(rows)])

    # --- projection instances (tests:test_acceptance.py:104-121 style) ---
    gen = np.random.default_rng(31)
    P, H, LO, IDX, SC, OUTP = [], [], [], [], [], []
    for _ in range(100):
        hi_r = gen.normal(size=(32, 8)).astype(np.float32)
        lo_r = gen.random((32, 2)).astype(np.float32)
        m = LandmarkModel.create(hi_r, lo_r)
        x = gen.normal(size=8).astype(np.float32)
        nbr = knn_base(x.reshape(1, -1), m.hi, 8)
        s = scores(nbr.sqdists[0])
        P.append(x); H.append(hi_r); LO.append(lo_r); IDX.append(nbr.indices[0]); SC.append(s.scores)
        OUTP.append(project_point(x, m, nbr.indices[0], s))
    arrays["proj_x"], arrays["proj_hi"], arrays["proj_lo"] = np.array(P), np.array(H), np.array(LO)
    arrays["proj_idx"], arrays["proj_scores"], arrays["proj_out"] = np.array(IDX), np.array(SC), np.array(OUTP)

    # --- degenerate layouts (tests:test_projection.py:98-105, 239-246) ---
    gen = np.random.default_rng(77)
    hi_d = gen.random((8, 3)).astype(np.float32)
    lo_d = np.zeros((8, 2), np.float32)
    lo_d[:4] = gen.random((4, 2))
    pts_d = gen.random((50, 3)).astype(np.float32)
    arrays["degen_hi"], arrays["degen_lo"], arrays["degen_points"] = hi_d, lo_d, pts_d
    arrays["degen_xy"] = embed(pts_d, LandmarkModel.create(hi_d, lo_d), EmbedParams(k=8))

    # --- C2/C3 shape: gaussians(16, 2^20, 32, seed=1), 16x16, k=16 (first 4096 rows) ---
    pts2, _ = rdg.gaussians(16, 1 << 20, 32, seed=1)
    hi2, lo2 = som_model(pts2, 16, 16, seed=2)
    sub = pts2[:4096]
    nb = knn_base(sub, hi2, 16)
    xy2 = project_neighbors(sub, LandmarkModel.create(hi2, lo2), nb)
    arrays["c2_idx"], arrays["c2_sqd"], arrays["c2_xy"] = nb.indices[:1024], nb.sqdists[:1024], xy2
    digests["c2"] = {"inputs": sha(pts2, hi2, lo2), "idx4096": sha(nb.indices), "sqd4096": sha(nb.sqdists)}
    # one online SOM tick (C3 trainer), sigma 1.0, alpha 0.1, batch 256
    ds2 = Dataset.from_points(pts2)
    m2 = LandmarkModel.create(hi2, lo2)
    rng = Rng(7)
    arrays["c3_som_sample"] = Rng(7).integers(0, ds2.n, size=256)
    arrays["c3_som_hi"] = som_tick(ds2, m2, SomConfig(sigma=1.0, alpha=0.1), rng)
    rng = Rng(8)
    arrays["c3_km_sample"] = Rng(8).integers(0, ds2.n, size=256)
    arrays["c3_km_hi"] = kmeans_tick(ds2, m2, KmeansConfig(), rng)
    del pts2, ds2
    print("c2/c3", time.time() - t0, flush=True)

    # --- C4 shape: gaussians(16, 10M, 32, seed=1), 32x32, k=16 (first 1024 rows) ---
    pts4, _ = rdg.gaussians(16, 10_000_000, 32, seed=1)
    hi4, lo4 = som_model(pts4, 32, 32, seed=2)
    sub = pts4[:1024].copy()
    nb = knn_base(sub, hi4, 16)
    xy4 = project_neighbors(sub, LandmarkModel.create(hi4, lo4), nb)
    arrays["c4_hi"], arrays["c4_lo"], arrays["c4_points"] = hi4, lo4, sub
    arrays["c4_idx"], arrays["c4_sqd"], arrays["c4_xy"] = nb.indices, nb.sqdists, xy4
    digests["c4"] = {"inputs_head": sha(pts4[:1 << 20]), "hi": sha(hi4)}
    del pts4
    print("c4", time.time() - t0, flush=True)

    # --- C5 shape: gaussians(32, 2^20, 512, seed=1), 64x64, k=32 (first 128 rows) ---
    pts5, _ = rdg.gaussians(32, 1 << 20, 512, seed=1)
    hi5, lo5 = som_model(pts5, 64, 64, seed=2)
    sub = pts5[:128].copy()
    nb = knn_base(sub, hi5, 32)
    xy5 = project_neighbors(sub, LandmarkModel.create(hi5, lo5), nb)
    arrays["c5_points"] = sub
    arrays["c5_idx"], arrays["c5_sqd"], arrays["c5_xy"] = nb.indices, nb.sqdists, xy5
    digests["c5"] = {"inputs_head": sha(pts5[:4096]), "hi": sha(hi5), "lo": sha(lo5)}
    del pts5
    print("c5", time.time() - t0, flush=True)

    # --- online trainers on the reference's small dataset (tests:conftest.py:17-21) ---
    gen = np.random.default_rng(11)
    small = gen.normal(size=(500, 5)).astype(np.float32)
    ds = Dataset.from_points(small)
    hi_s = small[Rng(1).choice_distinct(500, 16)]
    lo_s = lattice(4, 4)
    model = LandmarkModel.create(hi_s, lo_s)
    cfg = SomConfig(sigma=0.8, alpha=0.2, batch_size=64)
    rng = Rng(2)
    probe = Rng(2)
    his, samples = [], []
    for _ in range(5):
        samples.append(probe.integers(0, ds.n, size=64))
        model = model.with_hi(som_tick(ds, model, cfg, rng))
        his.append(model.hi.copy())
    arrays["small_points"], arrays["small_hi0"], arrays["small_lo"] = small, hi_s, lo_s
    arrays["small_som_samples"], arrays["small_som_his"] = np.array(samples), np.array(his)
    model = LandmarkModel.create(hi_s, lo_s)
    rng, probe = Rng(3), Rng(3)
    his, samples = [], []
    for _ in range(5):
        samples.append(probe.integers(0, ds.n, size=64))
        model = model.with_hi(kmeans_tick(ds, model, KmeansConfig(alpha_km=0.3, batch_size=64), rng))
        his.append(model.hi.copy())
    arrays["small_km_samples"], arrays["small_km_his"] = np.array(samples), np.array(his)
    arrays["small_qe"] = np.array([quantization_error(ds, hi_s)])

    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "digests.json").write_text(json.dumps(digests, indent=1, sort_keys=True))
    print("done", time.time() - t0, "s;", (OUT / "golden.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
