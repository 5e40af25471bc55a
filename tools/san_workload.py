"""Small workload that launches every hot kernel family once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
tc2 screen + BMU sort + exact (d = 32, g = 256 and 1024), projection
(reg2, reg3 records), tc3 GEMM screen + exact group (d = 512, g = 4096,
k = 32), online SOM / k-means ticks (row + cluster kernels), batch-SOM
statistics (shared-memory table and segment sums) + update, faithful
k-NN / scores / projection.

    python tools/san_workload.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2201_00701_b200 as esom  # noqa: E402
from paper_2201_00701_b200 import datagen  # noqa: E402
from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop  # noqa: E402

torch.cuda.set_device(0)
for rows, cols, n, d, k in ((16, 16, 1 << 14, 32, 16), (32, 32, 1 << 14, 32, 16), (64, 64, 2048, 512, 32)):
    pts = datagen.gaussians(16, n, d, seed=1)[0].astype(np.float32)
    hi, lo = datagen.som_model(pts, rows, cols, seed=2)
    X = torch.from_numpy(pts).cuda()
    model = esom.LandmarkModel.create(hi, lo)
    nb = esom.knn(X, torch.from_numpy(hi).cuda(), k)
    xy = esom.embed(X, model, esom.EmbedParams(k=k))
    xf = esom.embed(pts[:256], model, esom.EmbedParams(k=k), mode="faithful")
    if d <= 32:
        esom.som_tick(X, model, esom.SomConfig(), esom.Rng(3))
        esom.kmeans_tick(X, model, esom.KmeansConfig(), esom.Rng(4))
        loop = FrameLoop(X, hi, lo, k, BatchSomConfig(sigma=1.0, alpha=0.05))
        loop.frame()
    torch.cuda.synchronize()
    print(f"g={rows * cols} d={d} k={k}: knn {tuple(nb.indices.shape)}, embed ok", flush=True)
print("san workload done")
