"""Where the C2 end-to-end time goes: model preparation (host + device) vs
the chunked H2D / compute / D2H pipeline (esom.embed on a pinned tensor)."""
import statistics
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import make_inputs  # noqa: E402
import paper_2201_00701_b200 as esom  # noqa: E402
from paper_2201_00701_b200 import projection as P  # noqa: E402

dev = torch.device("cuda", 0)
pts, hi, lo, k, _, _ = make_inputs("c2", 0, 1)
host = torch.from_numpy(pts).pin_memory()
model = esom.LandmarkModel.create(hi, lo)
params = esom.EmbedParams(k=k)
for _ in range(3):
    esom.embed(host, model, params)
tp, tt = [], []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pm = P.PreparedModel(model.hi, model.lo, k, device=dev)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tp.append((t1 - t0, t2 - t0))
    t0 = time.perf_counter()
    esom.embed(host, model, params)
    tt.append(time.perf_counter() - t0)
print("prep host ms", round(1e3 * statistics.median(a for a, _ in tp), 3), "prep+sync ms",
      round(1e3 * statistics.median(b for _, b in tp), 3), "embed ms", round(1e3 * statistics.median(tt), 3),
      "ideal H2D ms", round(host.numel() * 4 / 52.2e9 * 1e3, 3))
for chunk in (1 << 16, 1 << 17, 1 << 18):
    P.PIPE_CHUNK = chunk
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        esom.embed(host, model, params)
        ts.append(time.perf_counter() - t0)
    print("chunk", chunk, "embed ms", round(1e3 * statistics.median(ts), 3))
