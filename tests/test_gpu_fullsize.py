"""Full-size parity at the north-star shapes: C4 = the whole
10M x 32 dataset against 1024 landmarks on ONE B200, and C5 = 2^20 x 512
against 4096 landmarks, k = 32 (the tensor-core GEMM screen).

Each shape is pinned three ways (pattern of ref tests/test_acceptance.py:37-67):
  * the dataset and model equal the reference's (sha256 of the generated
    head rows and of hi, recorded by running the reference: make_golden.py);
  * the head rows equal the reference's own knn_base / project_neighbors
    outputs (golden arrays), and a strided sample of every row range equals
    the C oracle bit for bit (k-NN) / to 1e-4 x extent (embedding);
  * size-independent properties on EVERY row, evaluated on the device:
    ascending distances, ties in index order, indices in range, nearest
    distance = the scan minimum, finite embeddings.
"""

import numpy as np
import pytest
import torch

from helpers import sha
from oracle import oracle
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen

pytestmark = pytest.mark.gpu


def _rows_properties(idx: torch.Tensor, sqd: torch.Tensor, g: int):
    """Every row: ascending, equal distances in index order, indices in [0, g), distinct."""
    dd = sqd[:, 1:] - sqd[:, :-1]
    assert bool((dd >= 0).all()), "distances not ascending"
    ties = dd == 0
    di = idx[:, 1:] - idx[:, :-1]
    assert bool((di[ties] > 0).all()), "equal distances not in index order"
    assert bool(((idx >= 0) & (idx < g)).all()), "index out of range"
    srt = torch.sort(idx, dim=1).values
    assert bool((srt[:, 1:] != srt[:, :-1]).all()), "duplicate neighbour"


def _sample_rows(n: int, step: int) -> np.ndarray:
    rows = np.arange(0, n, step)
    return np.unique(np.concatenate([rows, [n - 1]]))


def test_c4_full_10m_one_gpu(digests, golden):
    n, d, g, k = 10_000_000, 32, 1024, 16
    pts = datagen.gaussians_f32(16, n, d, seed=1)
    assert sha(pts[: 1 << 20]) == digests["c4"]["inputs_head"]
    hi, lo = datagen.som_model(pts, 32, 32, seed=2)
    assert sha(hi) == digests["c4"]["hi"]
    X = torch.from_numpy(pts).cuda()
    H = torch.from_numpy(hi).cuda()
    nb = esom.knn(X, H, k)
    idx, sqd = nb.indices, nb.sqdists
    # reference head (knn_base run by the reference on the first 1024 rows)
    assert np.array_equal(idx[:1024].cpu().numpy(), golden["c4_idx"])
    assert np.array_equal(sqd[:1024].cpu().numpy(), golden["c4_sqd"])
    # strided oracle sample across all 10M rows (bit-exact)
    rows = _sample_rows(n, 997)
    want_i, want_d = oracle.knn(pts[rows], hi, k)
    rt = torch.from_numpy(rows).cuda()
    assert np.array_equal(idx[rt].cpu().numpy(), want_i)
    assert np.array_equal(sqd[rt].cpu().numpy(), want_d)
    _rows_properties(idx, sqd, g)
    # the nearest distance of every row is the minimum over ALL landmarks:
    # x.x - 2 x.l + l.l in f64 on the device bounds the f32 sum's rounding
    nearest = torch.empty(n, dtype=torch.float64, device="cuda")
    Hd = H.double()
    hn = (Hd * Hd).sum(1)
    for s in range(0, n, 1 << 20):
        Xd = X[s:s + (1 << 20)].double()
        dm = (Xd * Xd).sum(1, keepdim=True) - 2.0 * Xd @ Hd.T + hn
        nearest[s:s + (1 << 20)] = dm.min(1).values
    err = (sqd[:, 0].double() - nearest).abs()
    assert bool((err <= 1e-4 * nearest.abs() + 1e-3).all()), float(err.max())
    del nb, idx, sqd, nearest
    # full-size embedding: the head against the reference's projection, a strided
    # sample against the oracle, every row finite
    model = esom.LandmarkModel.create(hi, lo)
    xy = esom.embed(X, model, esom.EmbedParams(k=k))
    assert bool(torch.isfinite(xy).all())
    ext = float(np.ptp(lo, axis=0).max())
    head = xy[:1024].cpu().numpy()
    assert float(np.abs(head - golden["c4_xy"]).max()) <= 1e-4 * ext
    ref = oracle.embed(pts[rows], hi, lo, k, threads=oracle.host_cores())
    assert float(np.abs(xy[rt].cpu().numpy() - ref).max()) <= 1e-4 * ext


def test_c5_full_size_tensor_core_screen(digests, golden):
    n, d, g, k = 1 << 20, 512, 4096, 32
    pts = datagen.gaussians_f32(32, n, d, seed=1)
    assert sha(pts[:4096]) == digests["c5"]["inputs_head"]
    hi, lo = datagen.som_model(pts, 64, 64, seed=2)
    assert sha(hi) == digests["c5"]["hi"] and sha(lo) == digests["c5"]["lo"]
    X = torch.from_numpy(pts).cuda()
    nb = esom.knn(X, torch.from_numpy(hi).cuda(), k)
    idx, sqd = nb.indices, nb.sqdists
    assert np.array_equal(idx[:128].cpu().numpy(), golden["c5_idx"])
    assert np.array_equal(sqd[:128].cpu().numpy(), golden["c5_sqd"])
    rows = _sample_rows(n, 4099)
    want_i, want_d = oracle.knn(pts[rows], hi, k)
    rt = torch.from_numpy(rows).cuda()
    assert np.array_equal(idx[rt].cpu().numpy(), want_i)
    assert np.array_equal(sqd[rt].cpu().numpy(), want_d)
    _rows_properties(idx, sqd, g)
    del nb, idx, sqd
    model = esom.LandmarkModel.create(hi, lo)
    xy = esom.embed(X, model, esom.EmbedParams(k=k))
    assert bool(torch.isfinite(xy).all())
    ext = float(np.ptp(lo, axis=0).max())
    assert float(np.abs(xy[:128].cpu().numpy() - golden["c5_xy"]).max()) <= 1e-4 * ext
    ref = oracle.embed(pts[rows], hi, lo, k, threads=oracle.host_cores())
    assert float(np.abs(xy[rt].cpu().numpy() - ref).max()) <= 1e-4 * ext
