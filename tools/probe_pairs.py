"""Probe: pair-table build time and bit-equality, tiled vs row-per-pair (ESOM_PAIR_V1)."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2201_00701_b200 as esom  # noqa: E402
from paper_2201_00701_b200 import datagen  # noqa: E402

torch.cuda.set_device(0)
for rows in (5, 16, 32, 64):
    pts = datagen.gaussians_f32(16, 1 << 16, 32, seed=1)
    hi, lo = datagen.som_model(pts, rows, rows + 1, seed=2)
    digests, times = [], []
    for v1 in (False, True):
        if v1:
            os.environ["ESOM_PAIR_V1"] = "1"
        else:
            os.environ.pop("ESOM_PAIR_V1", None)
        pm = esom.PreparedModel(hi, lo, 16)
        ts = []
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); pm.update(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        times.append(round(float(np.median(ts)), 4))
        digests.append(hashlib.sha256(pm.ws.cpu().numpy().tobytes()).hexdigest()[:16])
    print(rows * (rows + 1), "prepare ms tiled / v1", times, "workspace identical", digests[0] == digests[1], flush=True)
