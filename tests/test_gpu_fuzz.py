"""Randomised shapes across every k-NN / projection path (tensor-core screens,
GEMM screen, CUDA-core scan, sort path; reg2 / reg3 / fast projection), each
against the C oracle: k-NN bit-exact (indices AND squared distances), embed
within 1e-4 x extent.  Seeds are fixed, so a failure reproduces."""
import numpy as np
import pytest
import torch

from oracle import oracle
import paper_2201_00701_b200 as esom

pytestmark = pytest.mark.gpu


def _shapes():
    gen = np.random.default_rng(20261017)
    out = []
    for t in range(48):
        d = int(gen.choice([1, 2, 3, 5, 8, 13, 16, 24, 31, 32, 33, 40, 64, 96, 130]))
        g = int(gen.choice([4, 9, 31, 33, 64, 100, 255, 256, 257, 300, 513, 1000, 1024]
                           + ([1500, 2048, 4097] if t >= 24 else [])))
        k = int(gen.choice([3, 4, 5, 8, 12, 16, 20, 32, 48, 64]))
        k = min(k, g)
        n = int(gen.choice([1, 7, 100, 1500, 5000, 20000]))
        out.append((n, d, g, k, int(gen.integers(1 << 30))))
    return out


@pytest.mark.parametrize("n,d,g,k,seed", _shapes())
def test_fuzz_knn_and_embed(n, d, g, k, seed):
    gen = np.random.default_rng(seed)
    centers = gen.uniform(0, 10, size=(6, d))
    pts = (centers[gen.integers(0, 6, n)] + gen.normal(0, 0.5, size=(n, d))).astype(np.float32)
    hi = (centers[gen.integers(0, 6, g)] + gen.normal(0, 0.7, size=(g, d))).astype(np.float32)
    if g > 8:
        hi[3] = hi[2]  # duplicate landmark: equal-distance ties resolve by index
    lo = gen.uniform(0, 8, size=(g, 2)).astype(np.float32)
    X = torch.from_numpy(pts).cuda()
    nb = esom.knn_base(X, torch.from_numpy(hi).cuda(), k)
    wi, wd = oracle.knn(pts, hi, k)
    assert np.array_equal(nb.indices.cpu().numpy(), wi), (n, d, g, k)
    assert np.array_equal(nb.sqdists.cpu().numpy(), wd), (n, d, g, k)
    if k >= 3:
        xy = esom.embed(pts, esom.LandmarkModel.create(hi, lo), esom.EmbedParams(k=k), backend="base")
        ref = oracle.embed(pts, hi, lo, k, threads=oracle.host_cores())
        ext = float(np.ptp(lo, axis=0).max())
        assert np.abs(xy - ref).max() <= 1e-4 * ext, (n, d, g, k)
