"""k-NN parity on the B200: bit-exact indices AND squared distances against
the reference's own outputs (golden digests / arrays) and the CPU oracle."""
import numpy as np
import pytest
import torch

from helpers import c1_inputs, c2_inputs, grid_cells, grid_inputs, sha
from oracle import oracle
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen

pytestmark = pytest.mark.gpu


def test_c01_grid_bit_exact_full(digests):
    # tests:test_acceptance.py:37-67 -- all 180 cells at n = 10^4, both API backends
    for seed, d, g, k in grid_cells():
        p, l = grid_inputs(seed, d, g)
        ref = digests["c01_grid"][f"{seed}_{d}_{g}_{k}"]
        a = esom.knn_base(p, l, k)
        assert sha(a.indices) == ref["idx"], (seed, d, g, k)
        assert sha(a.sqdists) == ref["sqd"], (seed, d, g, k)
        if k in (4, 64):
            b = esom.knn_bitonic(p, l, k)
            assert np.array_equal(a.indices, b.indices) and np.array_equal(a.sqdists, b.sqdists)


def test_c1_bit_exact(golden):
    pts, hi, _ = c1_inputs()
    nb = esom.knn(pts, hi, 8)
    assert np.array_equal(nb.indices, golden["c1_idx"])
    assert np.array_equal(nb.sqdists, golden["c1_sqd"])


def test_sentinel_g257(golden):
    nb = esom.knn_bitonic(golden["sentinel257_points"], golden["sentinel257_landmarks"], 16)
    assert np.array_equal(nb.indices, golden["sentinel257_idx"])
    assert np.array_equal(nb.sqdists, golden["sentinel257_sqd"])


def test_known_answers(rng_np):
    lm = np.array([[0.0], [1.0], [2.0], [3.0]], np.float32)
    nb = esom.knn_base(np.array([[0.9]], np.float32), lm, 4)
    assert nb.indices[0].tolist() == [1, 0, 2, 3]
    np.testing.assert_allclose(nb.sqdists[0], [0.01, 0.81, 1.21, 4.41], rtol=1e-6)
    landmarks = rng_np.random((8, 3)).astype(np.float32)
    nb = esom.knn_base(landmarks[5:6], landmarks, 1)
    assert nb.indices[0, 0] == 5 and nb.sqdists[0, 0] == 0.0
    nb = esom.knn_base(np.array([[0.0]], np.float32), np.array([[1.0], [-1.0]], np.float32), 2)
    assert nb.indices[0].tolist() == [0, 1]
    same = np.tile(np.float32([1.5, -2.0]), (32, 1))
    nb = esom.knn_bitonic(rng_np.random((10, 2)).astype(np.float32), same, 8)
    assert np.array_equal(nb.indices, np.tile(np.arange(8, dtype=np.int32), (10, 1)))


@pytest.mark.parametrize("n,d,g,k", [(40, 6, 23, 7), (300, 5, 64, 3), (257, 1, 33, 5), (100, 3, 9, 9),
                                     (500, 7, 257, 64), (200, 12, 300, 100), (64, 2, 1000, 257),
                                     (1000, 48, 130, 31), (129, 100, 77, 10), (77, 513, 40, 12)])
def test_odd_shapes_vs_oracle(n, d, g, k):
    gen = np.random.default_rng(n * 7 + d)
    p = gen.normal(size=(n, d)).astype(np.float32)
    l = gen.normal(size=(g, d)).astype(np.float32)
    want_i, want_d = oracle.knn(p, l, k)
    nb = esom.knn_base(p, l, k)
    assert np.array_equal(nb.indices, want_i)
    assert np.array_equal(nb.sqdists, want_d)


def test_ties_and_duplicates():
    # many exact ties: integer lattice points against duplicated landmarks
    gen = np.random.default_rng(3)
    l = gen.integers(0, 3, size=(200, 4)).astype(np.float32)
    p = gen.integers(0, 3, size=(5000, 4)).astype(np.float32)
    for k in (4, 16, 33, 64):
        want_i, want_d = oracle.knn(p, l, k)
        nb = esom.knn_base(p, l, k)
        assert np.array_equal(nb.indices, want_i), k
        assert np.array_equal(nb.sqdists, want_d), k


def test_overflowing_distances_keep_reference_order():
    # finite inputs whose squared distances overflow to +inf (ref semantics:
    # the first k landmarks by index)
    p = np.array([[3e19, -3e19]], np.float32)
    l = np.array([[0.0, 0.0], [1.0, 1.0], [-1.0, 2.0], [5.0, 5.0], [1e19, 0.0]], np.float32)
    want_i, want_d = oracle.knn(p, l, 3)
    nb = esom.knn_base(p, l, 3)
    assert np.array_equal(nb.indices, want_i)
    assert np.array_equal(nb.sqdists, want_d)


def test_errors():
    with pytest.raises(esom.ParameterError):
        esom.knn_base(np.ones((2, 2)), np.ones((3, 2)), 4)
    with pytest.raises(esom.InputError):
        esom.knn_base(np.array([[np.inf, 0.0]], np.float32), np.ones((4, 2), np.float32), 2)
    with pytest.raises(esom.InputError):
        esom.knn_base(np.ones((3, 2), np.float32), np.array([[np.nan, 0.0]] * 4, np.float32), 2)
    with pytest.raises(esom.ParameterError):
        esom.knn_bitonic(np.ones((4, 2)), np.ones((32, 2)), 12)
    with pytest.raises(esom.ParameterError):
        esom.knn(np.ones((4, 2)), np.ones((8, 2)), 4, backend="carrier-pigeon")
    with pytest.raises(esom.InputError):
        esom.knn(np.ones((4, 3)), np.ones((8, 2)), 4)


def test_empty_and_device_tensors():
    nb = esom.knn_base(np.zeros((0, 4), np.float32), np.ones((8, 4), np.float32), 4)
    assert nb.indices.shape == (0, 4)
    gen = np.random.default_rng(5)
    p = gen.normal(size=(1000, 16)).astype(np.float32)
    l = gen.normal(size=(64, 16)).astype(np.float32)
    nbd = esom.knn(torch.from_numpy(p).cuda(), torch.from_numpy(l).cuda(), 16)
    assert nbd.indices.is_cuda
    want_i, want_d = oracle.knn(p, l, 16)
    assert np.array_equal(nbd.indices.cpu().numpy(), want_i)
    assert np.array_equal(nbd.sqdists.cpu().numpy(), want_d)


def test_c2_full_size(digests):
    # BASELINE configs[1] at full size (2^20 x 32, g = 256, k = 16): reference
    # digest on the first 4096 rows, oracle on a strided sample, and
    # size-independent properties on every row.
    pts, hi, _ = c2_inputs()
    nb = esom.knn(torch.from_numpy(pts).cuda(), torch.from_numpy(hi).cuda(), 16)
    idx = nb.indices.cpu().numpy()
    sqd = nb.sqdists.cpu().numpy()
    assert sha(idx[:4096]) == digests["c2"]["idx4096"]
    assert sha(sqd[:4096]) == digests["c2"]["sqd4096"]
    rows = np.arange(0, pts.shape[0], 97)
    want_i, want_d = oracle.knn(pts[rows], hi, 16)
    assert np.array_equal(idx[rows], want_i) and np.array_equal(sqd[rows], want_d)
    assert np.all(np.diff(sqd, axis=1) >= 0)
    ties = np.diff(sqd, axis=1) == 0
    assert np.all(np.diff(idx, axis=1)[ties] > 0)
    assert np.all((idx >= 0) & (idx < 256))


def test_c4_c5_heads(golden):
    nb = esom.knn(golden["c4_points"], golden["c4_hi"], 16)
    assert np.array_equal(nb.indices, golden["c4_idx"]) and np.array_equal(nb.sqdists, golden["c4_sqd"])
    pts5 = golden["c5_points"]
    hi5, _ = _c5_model()
    nb = esom.knn(pts5, hi5, 32)
    assert np.array_equal(nb.indices, golden["c5_idx"]) and np.array_equal(nb.sqdists, golden["c5_sqd"])


_C5 = None


def _c5_model():
    global _C5
    if _C5 is None:
        _C5 = datagen.som_model(datagen.gaussians_f32(32, 1 << 20, 512, seed=1), 64, 64, seed=2)
    return _C5
