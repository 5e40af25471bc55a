"""Pin the CPU oracle (oracle/esom_oracle.c) to the reference's own outputs.

Fixtures come from tests/golden/make_golden.py, which ran the reference
(`embedview`) in the build container.  Everything here is CPU-only.
"""
import math

import numpy as np
import pytest

from helpers import c1_inputs, c2_inputs, grid_cells, grid_inputs, sha
from oracle import oracle
from paper_2201_00701_b200 import datagen
from paper_2201_00701_b200.core import Rng


def test_datagen_reproduces_fixture_inputs(digests):
    pts, hi, lo = c1_inputs()
    assert sha(pts, hi, lo) == digests["c1"]["inputs"]
    for seed, d, g, k in list(grid_cells(ks=(4,)))[:6]:
        p, l = grid_inputs(seed, d, g)
        assert sha(p, l) == digests["c01_grid"][f"{seed}_{d}_{g}_{k}"]["inputs"]


def test_c2_inputs_match(digests):
    pts, hi, lo = c2_inputs()
    assert sha(pts, hi, lo) == digests["c2"]["inputs"]


@pytest.mark.parametrize("backend", ["base", "bitonic"])
def test_c1_knn_scores_embed_bit_exact(golden, backend):
    pts, hi, lo = c1_inputs()
    idx, sqd = oracle.knn(pts, hi, 8, backend)
    assert np.array_equal(idx, golden["c1_idx"])
    assert np.array_equal(sqd, golden["c1_sqd"])
    sc = oracle.scores(sqd)
    assert np.array_equal(sc, golden["c1_scores"])
    xy = oracle.embed(pts, hi, lo, 8, backend)
    assert np.array_equal(xy, golden["c1_xy"])


def test_c01_grid_subset_digests(digests):
    # tests:test_acceptance.py:37-67 (full grid runs in tests/test_gpu_knn.py)
    for seed, d, g, k in grid_cells(seeds=(101,), ds=(2, 16), gs=(16, 64, 257)):
        p, l = grid_inputs(seed, d, g)
        idx, sqd = oracle.knn(p, l, k)
        ref = digests["c01_grid"][f"{seed}_{d}_{g}_{k}"]
        assert sha(idx) == ref["idx"], (seed, d, g, k)
        assert sha(sqd) == ref["sqd"], (seed, d, g, k)
        if k in (4, 16):
            bi, bs = oracle.knn(p, l, k, "bitonic")
            assert np.array_equal(bi, idx) and np.array_equal(bs, sqd)


def test_sentinel_padding_g257(golden):
    idx, sqd = oracle.knn(golden["sentinel257_points"], golden["sentinel257_landmarks"], 16, "bitonic")
    assert np.array_equal(idx, golden["sentinel257_idx"])
    assert np.array_equal(sqd, golden["sentinel257_sqd"])


def test_known_answers():
    # tests:test_knn.py:36-40, 48-51
    lm = np.array([[0.0], [1.0], [2.0], [3.0]], np.float32)
    idx, sqd = oracle.knn(np.array([[0.9]], np.float32), lm, 4)
    assert idx[0].tolist() == [1, 0, 2, 3]
    np.testing.assert_allclose(sqd[0], [0.01, 0.81, 1.21, 4.41], rtol=1e-6)
    idx, _ = oracle.knn(np.array([[0.0]], np.float32), np.array([[1.0], [-1.0]], np.float32), 2)
    assert idx[0].tolist() == [0, 1]
    # tests:test_projection.py:59-69 closed form
    s = oracle.scores(np.array([0.0, 1.0, 4.0]))[0]
    np.testing.assert_allclose(s, [math.exp(0) - math.exp(-2), math.exp(-0.5) - math.exp(-2), 0.0], rtol=1e-12)


def test_scores_rows_bit_exact(golden):
    for i in range(int(golden["scores_count"][0])):
        got = oracle.scores(golden[f"scores_in_{i}"])[0]
        assert np.array_equal(got, golden[f"scores_out_{i}"]), i


def test_projection_instances_bit_exact(golden):
    for t in range(golden["proj_x"].shape[0]):
        out = oracle.project(golden["proj_x"][t:t + 1], golden["proj_hi"][t], golden["proj_lo"][t],
                             golden["proj_idx"][t:t + 1], golden["proj_scores"][t:t + 1])
        assert np.array_equal(out[0], golden["proj_out"][t]), t


def test_degenerate_layout_bit_exact(golden):
    xy = oracle.embed(golden["degen_points"], golden["degen_hi"], golden["degen_lo"], 8, "bitonic")
    assert np.array_equal(xy, golden["degen_xy"])
    assert np.all(np.isfinite(xy))


@pytest.mark.parametrize("case,k", [("c4", 16), ("c5", 32)])
def test_high_g_heads_bit_exact(golden, case, k):
    pts = golden[f"{case}_points"]
    if case == "c4":
        hi, lo = golden["c4_hi"], golden["c4_lo"]
    else:
        hi, lo = _c5_model()
    idx, sqd = oracle.knn(pts, hi, k)
    assert np.array_equal(idx, golden[f"{case}_idx"])
    assert np.array_equal(sqd, golden[f"{case}_sqd"])
    xy = oracle.project(pts, hi, lo, idx, oracle.scores(sqd))
    assert np.array_equal(xy, golden[f"{case}_xy"])


_C5 = None


def _c5_model():
    # regenerate the 64x64 model of gaussians(32, 2^20, 512, seed=1) (4 GB of
    # f64 normals); cached for the session
    global _C5
    if _C5 is None:
        pts = datagen.gaussians_f32(32, 1 << 20, 512, seed=1)
        _C5 = datagen.som_model(pts, 64, 64, seed=2)
    return _C5


def test_c2_head_bit_exact(golden, digests):
    pts, hi, lo = c2_inputs()
    sub = pts[:4096]
    idx, sqd = oracle.knn(sub, hi, 16)
    assert sha(idx) == digests["c2"]["idx4096"] and sha(sqd) == digests["c2"]["sqd4096"]
    xy = oracle.project(sub, hi, lo, idx, oracle.scores(sqd))
    assert np.array_equal(xy, golden["c2_xy"])


def _trainer_check(got, want, what):
    exact = float(np.mean(got == want))
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6, err_msg=what)
    return exact


def test_online_trainers_small(golden):
    pts, hi0, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    hi = hi0.copy()
    rng = Rng(2)
    for t in range(5):
        sample = rng.integers(0, pts.shape[0], size=64)
        assert np.array_equal(sample, golden["small_som_samples"][t])
        hi = oracle.som_tick(pts, hi, lo, sample, 0.8, 0.2)
        _trainer_check(hi, golden["small_som_his"][t], f"som tick {t}")
    hi = hi0.copy()
    for t in range(5):
        hi = oracle.kmeans_tick(pts, hi, golden["small_km_samples"][t], 0.3)
        _trainer_check(hi, golden["small_km_his"][t], f"kmeans tick {t}")
    assert oracle.quantization_error(pts, hi0) == pytest.approx(float(golden["small_qe"][0]), rel=1e-9)


def test_online_trainers_c3(golden):
    pts, hi, lo = c2_inputs()
    assert np.array_equal(Rng(7).integers(0, pts.shape[0], size=256), golden["c3_som_sample"])
    got = oracle.som_tick(pts, hi, lo, golden["c3_som_sample"], 1.0, 0.1)
    exact = _trainer_check(got, golden["c3_som_hi"], "c3 som")
    assert exact > 0.9
    got = oracle.kmeans_tick(pts, hi, golden["c3_km_sample"], 0.05)
    assert _trainer_check(got, golden["c3_km_hi"], "c3 kmeans") > 0.99


def test_batch_som_reduces_to_online_at_b1(golden):
    # SURVEY §8c T3 pin (ii): mean-field batch SOM with one sample == som_tick(batch 1)
    pts, hi0, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    for s in (3, 77, 401):
        online = oracle.som_tick(pts, hi0, lo, np.array([s]), 0.8, 0.4)
        batch = oracle.batch_som_step(pts[s:s + 1], hi0, lo, 0.8, 0.4)
        np.testing.assert_allclose(batch, online, rtol=1e-6, atol=1e-7)


def test_batch_som_properties(golden):
    pts, hi0, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    same = oracle.batch_som_step(pts, hi0, lo, 1.0, 0.0)
    assert np.array_equal(same, hi0)  # alpha = 0 leaves hi unchanged
    qe0 = oracle.quantization_error(pts, hi0)
    hi = hi0.copy()
    for t in range(20):
        hi = oracle.batch_som_step(pts, hi, lo, 1.5 + (0.3 - 1.5) * t / 19, 0.5)
    assert oracle.quantization_error(pts, hi) < qe0
