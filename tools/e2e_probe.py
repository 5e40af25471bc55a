"""End-to-end probe: pinned H2D / D2H bandwidth and esom.embed(pinned host)
wall time for the C2 workload under a few pipeline settings."""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import make_inputs  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    pts, hi, lo, k, _, _ = make_inputs("c2", 0, 1)
    host = torch.from_numpy(pts).pin_memory()
    d_buf = torch.empty(host.shape, dtype=torch.float32, device=dev)
    for _ in range(3):
        d_buf.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d_buf.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    h2d = host.numel() * 4 * 10 / (time.perf_counter() - t0) / 1e9
    out = torch.empty(host.shape, dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        out.copy_(d_buf, non_blocking=True)
    torch.cuda.synchronize()
    d2h = host.numel() * 4 * 10 / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"h2d_GBps": h2d, "d2h_GBps": d2h, "h2d_ms_per_step": host.numel() * 4 / h2d / 1e6}), flush=True)
    import importlib

    for chunk, depth in [(1 << 17, 3), (1 << 16, 4), (1 << 18, 3), (1 << 15, 6)]:
        os.environ["ESOM_PIPE_CHUNK"] = str(chunk)
        os.environ["ESOM_PIPE_DEPTH"] = str(depth)
        import paper_2201_00701_b200.projection as P
        importlib.reload(P)
        import paper_2201_00701_b200 as esom
        model = esom.LandmarkModel.create(hi, lo)
        params = esom.EmbedParams(k=k)
        P.embed(host, model, params)
        ts = []
        for _ in range(7):
            t0 = time.perf_counter()
            P.embed(host, model, params)
            ts.append(time.perf_counter() - t0)
        ms = statistics.median(ts) * 1e3
        print(json.dumps({"chunk": chunk, "depth": depth, "e2e_ms": ms, "Mpts_per_s": host.shape[0] / ms / 1e3}), flush=True)


if __name__ == "__main__":
    main()
