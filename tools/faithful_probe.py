"""Wall time of esom.embed(..., mode="faithful") on the C2 workload for a few
k (pairs per point = k(k-1)/2), and its kernel launch list under ncu
(python tools/faithful_probe.py [k ...])."""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import make_inputs  # noqa: E402
import paper_2201_00701_b200 as esom  # noqa: E402

pts, hi, lo, k0, _, _ = make_inputs("c2", 0, 1)
X = torch.from_numpy(pts).cuda()
model = esom.LandmarkModel.create(hi, lo)
for k in [int(a) for a in sys.argv[1:]] or [k0]:
    esom.embed(X, model, esom.EmbedParams(k=k), mode="faithful")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    esom.embed(X, model, esom.EmbedParams(k=k), mode="faithful")
    torch.cuda.synchronize()
    print("k", k, "pairs", k * (k - 1) // 2, "ms", round((time.perf_counter() - t0) * 1e3, 2), flush=True)
