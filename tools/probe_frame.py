"""One eager training frame (C3 / C4 shapes) after warm-up, for an ncu launch list:

    ncu --metrics gpu__time_duration.sum --csv python tools/probe_frame.py c3
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import make_inputs  # noqa: E402
from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
pts, hi, lo, k, train, n_total = make_inputs(wl, 0, 1)
X = torch.from_numpy(pts).cuda()
loop = FrameLoop(X, hi, lo, k, BatchSomConfig(sigma=1.0, alpha=0.05), train=train)
for _ in range(3):
    loop.frame()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("frame")
loop._eager_frame()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
