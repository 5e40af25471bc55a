"""Tensor-core k-NN probe: device time of esom_knn per screen variant
(ESOM_TC2_W = 2/3/4 warpgroups, 0 = round-streaming esom_tc.cuh, ESOM_TC=0
CUDA-core scan), bit-equality against the scan, and the mean number of
candidates re-evaluated exactly per point.

    python tools/tc_probe.py [c2 c4 ...]
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


def main(names):
    dev = torch.device("cuda", 0)
    L = _lib.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(8, dtype=torch.int32, device=dev)
    for name in names:
        pts, hi, lo, k, _, _ = make_inputs(name, 0, 1)
        n, d = pts.shape
        X = torch.from_numpy(pts).to(dev)
        H = torch.from_numpy(hi).to(dev)
        g = H.shape[0]
        ws = torch.empty(L.esom_workspace_bytes(g, d, k, 0), dtype=torch.uint8, device=dev)
        flag = _dev.new_flag(dev)
        st = _dev.stream_handle(dev)
        outs = {}
        for var in os.environ.get("PROBE_VARIANTS", "scan,w0,w2,w3,w4").split(","):
            os.environ["ESOM_TC"] = "0" if var == "scan" else "1"
            if var != "scan":
                os.environ["ESOM_TC2_W"] = var[1:]
            idx = torch.empty((n, k), dtype=torch.int32, device=dev)
            sqd = torch.empty((n, k), dtype=torch.float32, device=dev)

            def run():
                _lib.call("esom_knn", _dev.ptr(X), n, d, _dev.ptr(H), g, k, _dev.ptr(idx), _dev.ptr(sqd),
                          _dev.ptr(flag), _dev.ptr(ws), ws.numel(), st)
            ts = []
            for _ in range(6):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                run()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            cnt.zero_()
            L.esom_set_tc_stats(_dev.ptr(cnt))
            run()
            torch.cuda.synchronize()
            L.esom_set_tc_stats(None)
            outs[var] = (idx, sqd)
            same = (torch.equal(idx, outs["scan"][0]) and torch.equal(sqd, outs["scan"][1])) if "scan" in outs else None
            print(json.dumps({"shape": name, "variant": var, "ms": statistics.median(ts[1:]),
                              "Mpts_per_s": n / statistics.median(ts[1:]) / 1e3,
                              "cand_per_pt": int(cnt[0].item()) / n, "slow_pts": int(cnt[1].item()), "union_mean": int(cnt[2].item()) / max(1, int(cnt[3].item()) + int(cnt[4].item())), "groups": int(cnt[3].item()), "splits": int(cnt[4].item()), "bit_equal_scan": same}), flush=True)
        os.environ.pop("ESOM_TC2_W", None)
        os.environ.pop("ESOM_TC", None)
        del X, outs


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c4"])
