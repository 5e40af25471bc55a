"""Probe: cost of the pieces of one FrameEngine tick as the SOM trains
(embed time and screen candidates per point vs training ticks)."""
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen, _lib
torch.cuda.set_device(0)
pts = datagen.gaussians_f32(16, 1 << 20, 32, seed=1)
X = torch.from_numpy(pts).cuda()


def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))


eng = esom.FrameEngine(pts, seed=7, k=16, grid=(16, 16))
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
xy = torch.empty((X.shape[0], 2), device="cuda")
for tick in range(0, 41):
    if tick in (0, 1, 2, 5, 10, 20, 40):
        pm = esom.PreparedModel(eng.model.hi, eng.model.lo, 16)
        cnt.zero_()
        _lib.load().esom_set_tc_stats(cnt.data_ptr())
        pm.embed_into(X, xy); torch.cuda.synchronize()
        _lib.load().esom_set_tc_stats(None)
        h = eng.model.hi.astype(np.float64)
        d2 = ((h[:, None, :] - h[None, :, :]) ** 2).sum(-1) + np.eye(len(h)) * 1e30
        print(f"tick {tick}: embed {t(lambda: pm.embed_into(X, xy)):.3f} ms, candidates/pt {cnt.item() / X.shape[0]:.1f}, "
              f"min landmark sep {np.sqrt(d2.min()):.4f}, median nn sep {np.median(np.sqrt(d2.min(1))):.4f}", flush=True)
    eng.tick()
import ctypes
L = _lib.load()
pm = esom.PreparedModel(eng.model.hi, eng.model.lo, 16)
pm.embed_into(X, xy); torch.cuda.synchronize()
L.esom_timing_begin(1)
pm.embed_into(X, xy); torch.cuda.synchronize()
for name in ("knn_tc2_kernel", "knn_exact_bits_kernel", "project_kernel"):
    c = ctypes.c_int32(0)
    print(name, L.esom_timing_query(name.encode(), ctypes.byref(c)), c.value)
L.esom_timing_begin(0)
np.save("gpurun_out/som40_hi.npy", eng.model.hi); np.save("gpurun_out/som40_lo.npy", eng.model.lo)
