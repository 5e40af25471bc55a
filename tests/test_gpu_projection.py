"""Scores / projection / fused embed parity on the B200.

Tolerances (north_star): embeddings within max |xy - xy_ref| <= 1e-4 x the
embedding extent.  The faithful kernels are additionally held to bit-exact
on inputs that involve no exp (project_point with given scores) and report
the exact-row fraction where CUDA's exp may differ from glibc's by 1 ulp.
"""
import math

import numpy as np
import pytest
import torch

from helpers import c1_inputs, c2_inputs
from oracle import oracle
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen
from paper_2201_00701_b200.projection import ScoreVector

pytestmark = pytest.mark.gpu

TOL = 1e-4  # x extent


def extent(lo):
    lo = np.asarray(lo, np.float64)
    return float(max(lo[:, 0].max() - lo[:, 0].min(), lo[:, 1].max() - lo[:, 1].min(), 1e-30))


def assert_xy_close(got, want, lo, what=""):
    err = float(np.abs(got.astype(np.float64) - want.astype(np.float64)).max()) if len(got) else 0.0
    assert err <= TOL * extent(lo), f"{what}: max err {err:.3e} > {TOL} x extent {extent(lo):.3g}"
    return err / extent(lo)


def test_scores_rows(golden):
    worst = 0.0
    exact = 0
    cnt = int(golden["scores_count"][0])
    for i in range(cnt):
        got = esom.scores(golden[f"scores_in_{i}"]).scores
        want = golden[f"scores_out_{i}"]
        exact += int(np.array_equal(got, want))
        worst = max(worst, float(np.max(np.abs(got - want))))
    assert worst <= 1e-15, worst
    assert exact >= cnt * 0.5
    s = esom.scores(np.array([0.0, 1.0, 4.0])).scores
    np.testing.assert_allclose(s, [1 - math.exp(-2), math.exp(-0.5) - math.exp(-2), 0.0], rtol=1e-12)
    np.testing.assert_array_equal(esom.scores(np.full(5, 2.0)).scores, [1, 1, 1, 1, 0])
    with pytest.raises(esom.InputError):
        esom.scores(np.array([1.0, 0.5, 2.0]))


def test_project_point_bit_exact(golden):
    # scores are given -> no exp involved -> the faithful kernel is bit-exact
    for t in range(golden["proj_x"].shape[0]):
        model = esom.LandmarkModel.create(golden["proj_hi"][t], golden["proj_lo"][t])
        out = esom.project_point(golden["proj_x"][t], model, golden["proj_idx"][t],
                                 ScoreVector(scores=golden["proj_scores"][t]))
        assert np.array_equal(out, golden["proj_out"][t]), t


def test_c1_embed(golden):
    pts, hi, lo = c1_inputs()
    model = esom.LandmarkModel.create(hi, lo)
    fast = esom.embed(pts, model, esom.EmbedParams(k=8))
    rel = assert_xy_close(fast, golden["c1_xy"], lo, "c1 fast")
    faithful = esom.embed(pts, model, esom.EmbedParams(k=8), mode="faithful")
    assert_xy_close(faithful, golden["c1_xy"], lo, "c1 faithful")
    exact_rows = np.mean(np.all(faithful == golden["c1_xy"], axis=1))
    assert exact_rows > 0.9, exact_rows
    print(f"c1: fast max err/extent {rel:.2e}; faithful exact rows {exact_rows:.4f}")


def test_degenerate_layout_and_finite(golden):
    model = esom.LandmarkModel.create(golden["degen_hi"], golden["degen_lo"])
    for mode in ("fast", "faithful"):
        xy = esom.embed(golden["degen_points"], model, esom.EmbedParams(k=8), mode=mode)
        assert np.all(np.isfinite(xy))
        assert_xy_close(xy, golden["degen_xy"], golden["degen_lo"], mode)


def test_coincident_layout_falls_back_exactly(rng_np):
    hi = rng_np.random((8, 4)).astype(np.float32)
    lo = np.tile(np.float32([0.25, 0.75]), (8, 1))
    model = esom.LandmarkModel.create(hi, lo)
    x = rng_np.random((50, 4)).astype(np.float32)
    for mode in ("fast", "faithful"):
        xy = esom.embed(x, model, esom.EmbedParams(k=4), mode=mode)
        assert np.array_equal(xy, np.tile(lo[0], (50, 1))), mode


def test_fixed_point_c02():
    # tests:test_acceptance.py:70-77
    gen = np.random.default_rng(7)
    lo = gen.random((64, 2)).astype(np.float32)
    model = esom.LandmarkModel.create(lo, lo)
    pts = gen.random((1000, 2)).astype(np.float32)
    for mode in ("fast", "faithful"):
        out = esom.embed(pts, model, esom.EmbedParams(k=16), mode=mode)
        assert float(np.abs(out - pts).max()) <= 1e-4, mode


def test_equivariance_c04():
    # tests:test_acceptance.py:104-163 -- the reference's own instance stream
    # (default_rng(53), same draw order) through the device knn/scores/project_point
    gen = np.random.default_rng(53)
    worst = dict(scale=0.0, trans=0.0, rot=0.0, iso=0.0)
    for _ in range(100):
        hi = gen.normal(size=(24, 6)).astype(np.float32)
        lo = gen.random((24, 2)).astype(np.float32)
        model = esom.LandmarkModel.create(hi, lo)
        x = gen.normal(size=6).astype(np.float32)
        nb = esom.knn_base(x.reshape(1, -1), model.hi, 8)
        idx, s = nb.indices[0], esom.scores(nb.sqdists[0])
        base = esom.project_point(x, model, idx, s)
        c = float(gen.uniform(0.1, 10.0))
        worst["scale"] = max(worst["scale"], float(np.abs(
            esom.project_point(x, model, idx, ScoreVector(scores=s.scores * c)) - base).max()))
        t = gen.normal(size=2).astype(np.float32)
        worst["trans"] = max(worst["trans"], float(np.abs(
            esom.project_point(x, model.with_lo(model.lo + t), idx, s) - (base + t)).max()))
        th = float(gen.uniform(0, 2 * np.pi))
        rot = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        rl = (model.lo.astype(np.float64) @ rot.T).astype(np.float32)
        worst["rot"] = max(worst["rot"], float(np.abs(
            esom.project_point(x, model.with_lo(rl), idx, s) - base @ rot.T).max()))
        q, _ = np.linalg.qr(gen.normal(size=(6, 6)))
        shift = gen.normal(size=6)
        hi2 = (model.hi.astype(np.float64) @ q.T + shift).astype(np.float32)
        x2 = (x.astype(np.float64) @ q.T + shift).astype(np.float32)
        moved = model.with_hi(hi2)
        nb2 = esom.knn_base(x2.reshape(1, -1), moved.hi, 8)
        iso = esom.project_point(x2, moved, nb2.indices[0], esom.scores(nb2.sqdists[0]))
        worst["iso"] = max(worst["iso"], float(np.abs(iso - base).max()))
    ok = worst["scale"] <= 1e-6 and worst["trans"] <= 1e-5 and worst["rot"] <= 1e-5 and worst["iso"] <= 1e-4
    assert ok, worst


def test_chunking_and_backends_bit_identical(rng_np):
    pts = rng_np.random((10_000, 16)).astype(np.float32)
    hi = rng_np.normal(size=(256, 16)).astype(np.float32)
    lo = rng_np.random((256, 2)).astype(np.float32)
    model = esom.LandmarkModel.create(hi, lo)
    whole = esom.embed(pts, model, esom.EmbedParams(k=16))
    chunked = esom.embed(pts, model, esom.EmbedParams(k=16), chunk_size=1429)
    assert np.array_equal(whole, chunked)
    base = esom.embed(pts, model, esom.EmbedParams(k=16), backend="base")
    assert np.array_equal(whole, base)
    dup = esom.embed(np.tile(pts[:1], (5, 1)), model, esom.EmbedParams(k=16))
    assert np.all(dup == dup[0])
    want = oracle.embed(pts, hi, lo, 16)
    assert_xy_close(whole, want, lo, "random 10k")


@pytest.mark.parametrize("k", [3, 5, 8, 16, 32, 64])
def test_embed_k_sweep_vs_oracle(k):
    gen = np.random.default_rng(k)
    pts, _ = datagen.gaussians(6, 3000, 8, seed=k)
    hi = pts[gen.choice(3000, 100, replace=False)]
    lo = datagen.lattice(10, 10)
    model = esom.LandmarkModel.create(hi, lo)
    want = oracle.embed(pts, hi, lo, k)
    got = esom.embed(pts, model, esom.EmbedParams(k=k), backend="base")
    assert_xy_close(got, want, lo, f"k={k}")


def test_outliers_far_from_landmarks():
    # law-of-cosines guard: points 10..1000x farther than the landmark spacing
    gen = np.random.default_rng(11)
    hi = gen.normal(size=(64, 16)).astype(np.float32)
    lo = datagen.lattice(8, 8)
    far = (gen.normal(size=(2000, 16)) * np.repeat([10.0, 100.0, 1000.0, 1.0], 500)[:, None]).astype(np.float32)
    model = esom.LandmarkModel.create(hi, lo)
    want = oracle.embed(far, hi, lo, 16)
    got = esom.embed(far, model, esom.EmbedParams(k=16))
    assert_xy_close(got, want, lo, "outliers")


def test_c2_full_size_embed(golden):
    pts, hi, lo = c2_inputs()
    model = esom.LandmarkModel.create(hi, lo)
    xy = esom.embed(torch.from_numpy(pts).cuda(), model, esom.EmbedParams(k=16)).cpu().numpy()
    assert np.all(np.isfinite(xy))
    assert_xy_close(xy[:4096], golden["c2_xy"], lo, "c2 head vs reference")
    rows = np.arange(0, pts.shape[0], 211)
    want = oracle.embed(pts[rows], hi, lo, 16)
    assert_xy_close(xy[rows], want, lo, "c2 sample vs oracle")


def test_c4_c5_heads_embed(golden):
    model4 = esom.LandmarkModel.create(golden["c4_hi"], golden["c4_lo"])
    xy4 = esom.embed(golden["c4_points"], model4, esom.EmbedParams(k=16))
    assert_xy_close(xy4, golden["c4_xy"], golden["c4_lo"], "c4 head")
    from test_gpu_knn import _c5_model
    hi5, lo5 = _c5_model()
    xy5 = esom.embed(golden["c5_points"], esom.LandmarkModel.create(hi5, lo5), esom.EmbedParams(k=32))
    assert_xy_close(xy5, golden["c5_xy"], lo5, "c5 head")


def test_embed_errors(rng_np):
    model = esom.LandmarkModel.create(rng_np.normal(size=(8, 4)).astype(np.float32),
                                      rng_np.random((8, 2)).astype(np.float32))
    with pytest.raises(esom.ParameterError):
        esom.embed(rng_np.random((3, 4)), model, esom.EmbedParams(k=16), backend="bitonic")
    with pytest.raises(esom.InputError):
        esom.embed(rng_np.random((3, 5)), model, esom.EmbedParams(k=4))
    bad = rng_np.random((3, 4)).astype(np.float32)
    bad[1, 2] = np.nan
    with pytest.raises(esom.InputError):
        esom.embed(bad, model, esom.EmbedParams(k=4))


def test_host_pipeline_equals_device():
    # pinned host input takes the chunked H2D/compute/D2H pipeline; same rows out
    pts, hi, lo = c2_inputs()
    model = esom.LandmarkModel.create(hi, lo)
    host = torch.from_numpy(pts[:600_000].copy()).pin_memory()
    a = esom.embed(host, model, esom.EmbedParams(k=16))
    b = esom.embed(torch.from_numpy(pts[:600_000]).cuda(), model, esom.EmbedParams(k=16)).cpu().numpy()
    assert isinstance(a, np.ndarray) and np.array_equal(a, b)


@pytest.mark.parametrize("grid,k", [((16, 16), 16), ((32, 32), 16), ((16, 16), 32), ((16, 16), 8)])
def test_embed_on_trained_som_vs_oracle(grid, k):
    """A trained SOM packs the landmarks tightly in hi-space while points stay
    far from them (kappa = 2 max sqd max T in the hundreds to thousands): the
    projection must keep the tolerance there without the exact f64 pair loop
    (f64 neighbour distances as offsets, esom_project.cuh precise_sqd)."""
    pts = datagen.gaussians(16, 1 << 15, 32, seed=1)[0].astype(np.float32)
    eng = esom.FrameEngine(pts, seed=7, k=16, grid=grid)
    for _ in range(12):
        eng.tick()
    hi, lo = eng.model.hi, eng.model.lo
    model = esom.LandmarkModel.create(hi, lo)
    xy = esom.embed(pts, model, esom.EmbedParams(k=k))
    ref = oracle.embed(pts, hi, lo, k, threads=oracle.host_cores())
    assert_xy_close(xy, ref, lo, f"trained {grid} k={k}")
    if grid != (16, 16) or k != 16:
        return
    # the far-point regime is really exercised (C3 shape)
    h = hi.astype(np.float64)
    hd2 = ((h[:, None, :] - h[None, :, :]) ** 2).sum(-1)[np.triu_indices(len(h), 1)]
    _, sqd = oracle.knn(pts[:2000], hi, k)
    assert np.median(2 * sqd.max(1) * 0.5 / hd2.min()) > 256


def test_embed_beyond_fast_kernel_shapes_falls_back():
    """g beyond the fast projection's shared-memory plan (k = 64: g > ~11k):
    embed falls back to the faithful chain instead of failing, as the
    reference handles any g (numpy, pinned-host and device inputs)."""
    gen = np.random.default_rng(9)
    g, d, k = 12_288, 8, 64
    hi = gen.normal(size=(g, d)).astype(np.float32)
    lo = gen.uniform(0, 100, size=(g, 2)).astype(np.float32)
    pts = gen.normal(size=(600, d)).astype(np.float32)
    model = esom.LandmarkModel.create(hi, lo)
    want = oracle.embed(pts, hi, lo, k)
    ext = float(np.ptp(lo, axis=0).max())
    for inp in (pts, torch.from_numpy(pts).cuda()):
        got = esom.embed(inp, model, esom.EmbedParams(k=k))
        got = got.cpu().numpy() if isinstance(got, torch.Tensor) else got
        assert float(np.abs(got - want).max()) <= 1e-4 * ext


def test_projection_system_matches_reference_formula(golden):
    """projection_system (ref: projection.py:151-186): the f64 normal equations;
    their Cramer solution is the faithful projection of the same point, and A
    is symmetric positive semi-definite."""
    pts, hi, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    model = esom.LandmarkModel.create(hi, lo)
    nb = esom.knn_base(pts[:50], hi, 8)
    for i in range(50):
        s = esom.scores(nb.sqdists[i])
        a, c = esom.projection_system(pts[i], model, nb.indices[i], s)
        assert np.allclose(a, a.T) and np.all(np.linalg.eigvalsh(a) >= -1e-9)
        det = a[0, 0] * a[1, 1] - a[0, 1] ** 2
        tr = a[0, 0] + a[1, 1]
        xy = esom.project_point(pts[i], model, nb.indices[i], s)
        if det >= 1e-9 * tr * tr + 1e-30:
            sol = np.array([(c[0] * a[1, 1] - c[1] * a[0, 1]) / det, (a[0, 0] * c[1] - a[0, 1] * c[0]) / det])
            assert np.allclose(sol.astype(np.float32), xy, rtol=1e-5, atol=1e-5 * float(np.ptp(lo)))


def test_numpy_input_pinned_in_place_on_reuse():
    """embed(numpy) through the chunked host pipeline: the first call stages the
    rows through pinned chunks, a repeated call pins the caller's array in
    place (cudaHostRegister) and DMAs from it; results identical, and the
    range is released when the array is collected."""
    import gc

    from paper_2201_00701_b200 import projection as P

    pts, hi, lo = c2_inputs()
    x = np.array(pts[: 1 << 19])  # a fresh owning array (8 MiB+)
    model = esom.LandmarkModel.create(hi, lo)
    params = esom.EmbedParams(k=16)
    a = esom.embed(x, model, params)
    n0 = len(P._HOST_REG)
    b = esom.embed(x, model, params)
    c = esom.embed(x, model, params)
    assert len(P._HOST_REG) == n0 + 1
    assert np.array_equal(a, b) and np.array_equal(a, c)
    want = esom.embed(torch.from_numpy(pts[: 1 << 19]).cuda(), model, params).cpu().numpy()
    assert np.array_equal(a, want)
    del x
    gc.collect()
    assert len(P._HOST_REG) == n0


@pytest.mark.parametrize("rows,cols,n", [(16, 16, 300_000), (12, 12, 70_001)])
def test_fused_exact_projection_equals_two_kernel_path(rows, cols, n):
    """embed's fused exact-k-NN + projection kernel (esom_fused.cuh, k = 16, the
    pair triangle in shared memory) gives the SAME bits as the two-kernel path
    (forced here by the nearest-landmark visiting order, which never fuses)."""
    from paper_2201_00701_b200.projection import PreparedModel

    pts = datagen.gaussians(16, n, 32, seed=3)[0].astype(np.float32)
    hi, lo = datagen.som_model(pts, rows, cols, seed=4)
    X = torch.from_numpy(pts).cuda()
    pm = PreparedModel(hi, lo, 16)
    a = torch.empty((n, 2), dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    pm.embed_into(X, a)
    pm.embed_into(X, b, bmu_order=True)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    want = oracle.embed(pts[::997], hi, lo, 16)
    ext = float(np.ptp(lo, axis=0).max())
    assert float(np.abs(a[::997].cpu().numpy() - want).max()) <= 1e-4 * ext


@pytest.mark.parametrize("d", [4, 8, 24, 32, 48, 64, 512])
def test_faithful_projection_paths_bit_exact(d):
    """The faithful projection kernel (ref: projection.py:68-121) takes a
    register-resident path for d <= 32 and 256-bit row loads for d % 8 == 0
    (else the generic loop): with the scores given (no exp involved) every
    path equals the C oracle's restatement bit for bit."""
    from paper_2201_00701_b200.projection import _project_dev
    gen = np.random.default_rng(100 + d)
    g, k, n = 80, 12, 600
    hi = (gen.normal(size=(g, d)) * 3).astype(np.float32)
    lo = (gen.random((g, 2)) * 10).astype(np.float32)
    pts = (gen.normal(size=(n, d)) * 3).astype(np.float32)
    idx = np.stack([gen.choice(g, k, replace=False) for _ in range(n)]).astype(np.int32)
    sc = np.sort(gen.random((n, k)), axis=1)[:, ::-1].copy()
    sc[:, -1] = 0.0
    sc[::7, 3] = 0.0  # zero-score neighbours are skipped like the reference's
    want = oracle.project(pts, hi, lo, idx, sc)
    got = _project_dev(torch.from_numpy(pts).cuda(), torch.from_numpy(hi).cuda(), torch.from_numpy(lo).cuda(),
                       torch.from_numpy(idx).cuda(), torch.from_numpy(sc).cuda()).cpu().numpy()
    assert np.array_equal(got, want), float(np.abs(got - want).max())
