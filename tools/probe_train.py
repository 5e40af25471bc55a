"""Probe: online trainer tick time (device) for the C3 / C4 shapes, on-chip
cluster kernel vs the global-memory kernel (ESOM_TICK_GLOBAL=1)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2201_00701_b200 as esom  # noqa: E402
from paper_2201_00701_b200 import datagen  # noqa: E402
from paper_2201_00701_b200.core import Rng  # noqa: E402

torch.cuda.set_device(0)
pts = datagen.gaussians_f32(16, 1 << 20, 32, seed=1)
X = torch.from_numpy(pts).cuda()


class D:
    points = X


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for rows, cols in ((16, 16), (32, 32), (64, 64)):
    hi, lo = datagen.som_model(pts, rows, cols, seed=2)
    model = esom.LandmarkModel.create(hi, lo)
    rng = Rng(3)
    ms = t(lambda: esom.som_tick(D, model, esom.SomConfig(), rng))
    km = t(lambda: esom.kmeans_tick(D, model, esom.KmeansConfig(), rng))
    print(f"g={rows * cols}: som_tick {ms:.3f} ms, kmeans_tick {km:.3f} ms (256 samples)", flush=True)

# kernel alone through the C ABI (device buffers prepared up front)
from paper_2201_00701_b200 import _dev, _lib  # noqa: E402

for rows, cols in ((16, 16), (32, 32)):
    hi, lo = datagen.som_model(pts, rows, cols, seed=2)
    g, d = hi.shape
    H = torch.from_numpy(hi).cuda()
    Lo = torch.from_numpy(lo).cuda()
    ws = torch.empty(_lib.load().esom_tick_workspace_bytes(g, d), dtype=torch.uint8, device="cuda")
    st = _dev.stream_handle(torch.device("cuda"))
    for B in (1, 16, 256):
        S = torch.randint(0, X.shape[0], (B,), dtype=torch.int64, device="cuda")
        ms = t(lambda: _lib.call("esom_som_tick", _dev.ptr(X), d, _dev.ptr(S), B, _dev.ptr(H), _dev.ptr(Lo), g, 1.0,
                                 0.1, _dev.ptr(ws), ws.numel(), st), reps=10)
        print(f"g={g} B={B}: esom_som_tick kernel {ms * 1e3:.1f} us", flush=True)
