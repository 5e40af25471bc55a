"""Kernel launch list of one esom.embed(..., mode="faithful") call on the C2
workload (run under ncu --metrics gpu__time_duration.sum)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import make_inputs  # noqa: E402
import paper_2201_00701_b200 as esom  # noqa: E402

pts, hi, lo, k, _, _ = make_inputs("c2", 0, 1)
X = torch.from_numpy(pts).cuda()
model = esom.LandmarkModel.create(hi, lo)
esom.embed(X, model, esom.EmbedParams(k=k), mode="faithful")
torch.cuda.synchronize()
