"""Multi-rank paths on ONE B200 (two processes sharing cuda:0, gloo carrying
the CUDA-tensor collectives; on a multi-GPU node the same calls go over
NCCL): the batch-SOM FrameLoop over row shards and the sharded online ticks
must reproduce the single-rank results."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import paper_2201_00701_b200 as esom
    from paper_2201_00701_b200 import datagen
    from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop
    from paper_2201_00701_b200.core import Rng
    from paper_2201_00701_b200.sharded import som_tick_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pts = datagen.gaussians(16, 100_000, 32, seed=1)[0].astype(np.float32)
    hi, lo = datagen.som_model(pts, 16, 16, seed=2)
    bounds = np.linspace(0, len(pts), world + 1).astype(int)
    X = torch.from_numpy(pts[bounds[rank]:bounds[rank + 1]]).cuda()
    loop = FrameLoop(X, hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
    for _ in range(5):
        loop.frame()
    model = esom.LandmarkModel.create(hi, lo)
    h_online = som_tick_sharded(X, int(bounds[rank]), len(pts), model, esom.SomConfig(), Rng(9))
    torch.cuda.synchronize()
    np.save(Path(out_dir) / f"batch{rank}.npy", loop.model.hi.cpu().numpy())
    np.save(Path(out_dir) / f"online{rank}.npy", h_online.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_match_single_rank(tmp_path):
    import torch.multiprocessing as mp

    import paper_2201_00701_b200 as esom
    from paper_2201_00701_b200 import datagen
    from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop
    from paper_2201_00701_b200.core import Rng

    port = 31500 + (os.getpid() % 1000)
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    b0, b1 = np.load(tmp_path / "batch0.npy"), np.load(tmp_path / "batch1.npy")
    o0, o1 = np.load(tmp_path / "online0.npy"), np.load(tmp_path / "online1.npy")
    assert np.array_equal(b0, b1) and np.array_equal(o0, o1)  # replicas stay identical
    pts = datagen.gaussians(16, 100_000, 32, seed=1)[0].astype(np.float32)
    hi, lo = datagen.som_model(pts, 16, 16, seed=2)
    X = torch.from_numpy(pts).cuda()
    loop = FrameLoop(X, hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
    for _ in range(5):
        loop.frame()
    # exact int64 fixed-point statistics: 5 training frames over two row shards give
    # landmarks bit-identical to one rank holding every point (SURVEY §7 hard part 6)
    assert np.array_equal(b0, loop.model.hi.cpu().numpy())
    online = esom.som_tick(X, esom.LandmarkModel.create(hi, lo), esom.SomConfig(), Rng(9)).cpu().numpy()
    assert np.array_equal(o0, online)  # the gathered sample rows are bit-exact
