"""Reproduce one fuzz case (tests/test_gpu_fuzz.py) with per-point errors and path switches."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle  # noqa: E402
import paper_2201_00701_b200 as esom  # noqa: E402

n, d, g, k, seed = map(int, sys.argv[1:6])
gen = np.random.default_rng(seed)
centers = gen.uniform(0, 10, size=(6, d))
pts = (centers[gen.integers(0, 6, n)] + gen.normal(0, 0.5, size=(n, d))).astype(np.float32)
hi = (centers[gen.integers(0, 6, g)] + gen.normal(0, 0.7, size=(g, d))).astype(np.float32)
if g > 8:
    hi[3] = hi[2]
lo = gen.uniform(0, 8, size=(g, 2)).astype(np.float32)
ref = oracle.embed(pts, hi, lo, k)
for mode in ("fast", "faithful"):
    xy = esom.embed(pts, esom.LandmarkModel.create(hi, lo), esom.EmbedParams(k=k), backend="base", mode=mode)
    err = np.abs(xy - ref).max(axis=1)
    print(mode, "max err", err.max(), "per point", np.round(err, 5))
idx, sqd = oracle.knn(pts, hi, k)
print("idx", idx[int(np.argmax(err))], "sqd", sqd[int(np.argmax(err))])
