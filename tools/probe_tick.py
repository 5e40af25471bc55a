"""Probe: embed cost (per kernel) as an online SOM trains (FrameEngine on C3 data).
A trained SOM packs landmarks tightly in hi-space; this is where the projection's
far-point handling matters (esom_project.cuh precise_sqd)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2201_00701_b200 as esom  # noqa: E402
from paper_2201_00701_b200 import _lib, datagen  # noqa: E402

torch.cuda.set_device(0)
grid = (32, 32) if "g1024" in sys.argv else (16, 16)
pts = datagen.gaussians_f32(16, 1 << 20, 32, seed=1)
X = torch.from_numpy(pts).cuda()
L = _lib.load()
eng = esom.FrameEngine(pts, seed=7, k=16, grid=grid)
xy = torch.empty((X.shape[0], 2), device="cuda")
for tick in range(0, 41):
    if tick in (0, 2, 10, 40):
        pm = esom.PreparedModel(eng.model.hi, eng.model.lo, 16)
        pm.embed_into(X, xy)
        torch.cuda.synchronize()
        L.esom_timing_begin(1)
        pm.embed_into(X, xy)
        torch.cuda.synchronize()
        ks = {}
        for name in ("knn_tc2_kernel", "knn_exact_bits_kernel", "project_kernel"):
            c = ctypes.c_int32(0)
            ks[name] = round(L.esom_timing_query(name.encode(), ctypes.byref(c)), 4)
        L.esom_timing_begin(0)
        print(f"grid {grid} tick {tick}: {ks}", flush=True)
    eng.tick()
