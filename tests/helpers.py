"""Shared test helpers (inputs regenerated from the reference's seeds)."""
import hashlib

import numpy as np

from paper_2201_00701_b200 import datagen


def sha(*arrays) -> str:
    """Same digest as tests/golden/make_golden.py:sha."""
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def c1_inputs():
    pts, _ = datagen.gaussians(8, 10_000, 4, seed=1)
    hi, lo = datagen.som_model(pts, 8, 8, seed=2)
    return pts, hi, lo


def c2_inputs():
    pts, _ = datagen.gaussians(16, 1 << 20, 32, seed=1)
    hi, lo = datagen.som_model(pts, 16, 16, seed=2)
    return pts, hi, lo


def small_inputs(golden):
    return golden["small_points"], golden["small_hi0"], golden["small_lo"]


def grid_cells(seeds=(101, 202, 303), ds=(2, 16, 64), gs=(16, 64, 257, 1024), ks=(4, 8, 16, 32, 64)):
    for seed in seeds:
        for d in ds:
            for g in gs:
                for k in ks:
                    if k <= g:
                        yield seed, d, g, k


def grid_inputs(seed, d, g):
    return datagen.uniform(10_000, d, seed), datagen.uniform(g, d, seed + g)
