"""Per-kernel device times for the BASELINE shapes (CUDA events, warm, L2 flushed).

    python tools/kernel_times.py [c2 c4 c5 ...]

Prints one JSON line per shape: k-NN scan alone, full embed (scan +
projection), their difference (projection), and points/s.
"""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import WORKLOADS, make_inputs  # noqa: E402
from paper_2201_00701_b200 import _dev, _lib  # noqa: E402
from paper_2201_00701_b200.projection import PreparedModel  # noqa: E402


def timed(fn, flush, reps=7):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[1:])


def main(names):
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    L = _lib.load()
    for name in names:
        pts, hi, lo, k, _, _ = make_inputs(name, 0, 1)
        n, d = pts.shape
        X = torch.from_numpy(pts).to(dev)
        pm = PreparedModel(hi, lo, k, device=dev)
        g = pm.g
        idx = torch.empty((n, k), dtype=torch.int32, device=dev)
        sqd = torch.empty((n, k), dtype=torch.float32, device=dev)
        flag = _dev.new_flag(dev)
        ws = torch.empty(L.esom_workspace_bytes(g, d, k, 0), dtype=torch.uint8, device=dev)
        st = _dev.stream_handle(dev)

        def knn():
            _lib.call("esom_knn", _dev.ptr(X), n, d, _dev.ptr(pm.hi), g, k, _dev.ptr(idx), _dev.ptr(sqd),
                      _dev.ptr(flag), _dev.ptr(ws), ws.numel(), st)

        xy = torch.empty((n, 2), dtype=torch.float32, device=dev)

        def embed():
            pm.embed_into(X, xy)

        def prep():
            pm.update()

        import os
        os.environ["ESOM_TC"] = "0"
        t_scan = timed(knn, flush)
        os.environ["ESOM_TC"] = "1"
        t_knn = timed(knn, flush)
        t_emb = timed(embed, flush)
        t_prep = timed(prep, flush)
        print(json.dumps({"shape": name, "n": n, "d": d, "g": g, "k": k, "knn_scan_ms": t_scan, "knn_ms": t_knn,
                          "embed_ms": t_emb, "projection_ms": t_emb - t_knn, "prepare_model_ms": t_prep,
                          "embed_Mpts_per_s": n / t_emb / 1e3}), flush=True)
        del X, idx, sqd, xy, pm


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c4"])
