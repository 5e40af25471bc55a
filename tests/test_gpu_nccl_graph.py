"""The multi-GPU training frame as ONE CUDA graph: FrameLoop.capture() records
the embed + BMU statistics, the NCCL all-reduce of the int64 statistics and
the landmark update.  Only one GPU is available here, so this runs a 1-rank
NCCL communicator with the all-reduce forced on (a rank-count-1 collective
still launches NCCL's kernel): capture must succeed, replays must equal
eager frames bit for bit, and NCCL must report its communicator init
(bench.py runs N > 1 this way, NCCL_DEBUG=INFO in its stderr)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist
from paper_2201_00701_b200 import batch_som, datagen
from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
pts = datagen.gaussians(16, 200_000, 32, seed=1)[0].astype(np.float32)
hi, lo = datagen.som_model(pts, 16, 16, seed=2)
X = torch.from_numpy(pts).cuda()
eager = FrameLoop(X, hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
for _ in range(4):
    eager.frame()
calls = []
def forced(buf, group=None):
    calls.append(buf.numel())
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
batch_som._allreduce_ = forced
g = FrameLoop(X, hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
g.frame()          # eager frame 1 (census)
g.capture()        # eager frame 2, then the recorded frame (not executed)
g.frame(); g.frame()  # replays: frames 3 and 4
torch.cuda.synchronize()
assert calls, "all-reduce never issued"
assert torch.equal(eager.model.hi, g.model.hi), "graph replay with NCCL differs from eager"
assert torch.equal(eager.xy, g.xy)
print("OK graph_launches", g.graph_launches, "allreduce_calls", len(calls))
dist.destroy_process_group()
"""


def test_frame_graph_captures_nccl_allreduce(tmp_path):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(32500 + os.getpid() % 1000),
               NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "OK graph_launches" in r.stdout
    assert "NCCL INFO" in r.stdout + r.stderr  # the communicator came up through NCCL
