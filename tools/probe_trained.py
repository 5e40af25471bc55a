"""Probe: per-kernel device times of one C2 frame on the initial and on a
trained model (T online SOM ticks), through FrameLoop (census-chosen visiting
order), for ncu captures of the trained projection.

    python tools/probe_trained.py [ticks] [workload] [only]
"""
import ctypes
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import WORKLOADS, make_inputs, train_model  # noqa: E402
from paper_2201_00701_b200 import _lib  # noqa: E402
from paper_2201_00701_b200.batch_som import FrameLoop  # noqa: E402

ticks = int(sys.argv[1]) if len(sys.argv) > 1 else 40
wl = sys.argv[2] if len(sys.argv) > 2 else "c2"
dev = torch.device("cuda", 0)
pts, hi, lo, k, train, n_total = make_inputs(wl, 0, 1)
X = torch.from_numpy(pts).to(dev)
L = _lib.load()
only = len(sys.argv) > 3 and sys.argv[3] == "only"  # the trained model alone (ncu captures)
for t in ((ticks,) if only else (0, ticks)):
    h = train_model(X, hi, lo, t, 1) if t else hi
    loop = FrameLoop(X, h, lo, k, train=False)
    for _ in range(3):
        loop.frame()
    torch.cuda.synchronize()
    L.esom_timing_begin(1)
    loop._eager_frame()
    torch.cuda.synchronize()
    out = {}
    for name in ("knn_tc2_kernel", "knn_exact_bits_kernel", "embed_fused_kernel", "project_kernel", "knn_gemm_kernel",
                 "knn_exact_group_kernel"):
        c = ctypes.c_int32(0)
        ms = L.esom_timing_query(name.encode(), ctypes.byref(c))
        if c.value:
            out[name] = round(ms, 4)
    L.esom_timing_begin(0)
    cnt = torch.zeros(8, dtype=torch.int32, device=dev)
    L.esom_set_tc_stats(cnt.data_ptr())
    loop._eager_frame()
    torch.cuda.synchronize()
    L.esom_set_tc_stats(None)
    print(json.dumps({"workload": wl, "ticks": t, "bmu_order": loop.bmu_order, "kernels_ms": out,
                      "cand_per_pt": int(cnt[0].item()) / X.shape[0], "slow_pts": int(cnt[1].item())}), flush=True)
