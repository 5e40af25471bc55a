"""C5 probe: k-NN device time of the GEMM-screen variants (env switches read
at launch), candidate counts, bit-equality against the default variant.

    python tools/probe_c5.py [VAR=VAL,VAR=VAL ...]   (each arg = one variant)
"""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import make_inputs  # noqa: E402
from paper_2201_00701_b200 import _dev, _lib  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
cnt = torch.zeros(8, dtype=torch.int32, device=dev)
pts, hi, lo, k, _, _ = make_inputs("c5", 0, 1)
n, d = pts.shape
X = torch.from_numpy(pts).to(dev)
H = torch.from_numpy(hi).to(dev)
g = H.shape[0]
ws = torch.empty(L.esom_workspace_bytes(g, d, k, 0), dtype=torch.uint8, device=dev)
flag = _dev.new_flag(dev)
st = _dev.stream_handle(dev)
ref = None
for spec in ["default"] + sys.argv[1:]:
    env = {} if spec == "default" else dict(kv.split("=") for kv in spec.split(","))
    os.environ.update(env)
    idx = torch.empty((n, k), dtype=torch.int32, device=dev)
    sqd = torch.empty((n, k), dtype=torch.float32, device=dev)

    def run():
        _lib.call("esom_knn", _dev.ptr(X), n, d, _dev.ptr(H), g, k, _dev.ptr(idx), _dev.ptr(sqd), _dev.ptr(flag),
                  _dev.ptr(ws), ws.numel(), st)

    ts = []
    for _ in range(4):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    L.esom_timing_begin(1)
    run()
    torch.cuda.synchronize()
    kt = {}
    import ctypes
    for name in ("knn_gemm_kernel", "knn_exact_group_kernel", "knn_exact_stage_kernel"):
        c = ctypes.c_int32(0)
        ms = L.esom_timing_query(name.encode(), ctypes.byref(c))
        if c.value:
            kt[name] = round(ms, 3)
    L.esom_timing_begin(0)
    cnt.zero_()
    L.esom_set_tc_stats(_dev.ptr(cnt))
    run()
    torch.cuda.synchronize()
    L.esom_set_tc_stats(None)
    if ref is None:
        ref = (idx, sqd)
    same = torch.equal(idx, ref[0]) and torch.equal(sqd, ref[1])
    print(json.dumps({"variant": spec, "ms": statistics.median(ts[1:]), "kernels": kt,
                      "cand_per_pt": int(cnt[0].item()) / n, "slow_pts": int(cnt[1].item()), "stats": cnt.tolist(),
                      "bit_equal_default": same}), flush=True)
    for key in env:
        os.environ.pop(key)
