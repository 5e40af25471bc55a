"""Landmark training on the B200: online SOM / k-means vs the reference's
goldens (f64 internally; only exp ulps and exact BMU near-ties may differ),
batch SOM vs the oracle restatement, and the reference's trainer properties."""
import numpy as np
import pytest
import torch

from helpers import c2_inputs
from oracle import oracle
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen
from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop, batch_som_step
from paper_2201_00701_b200.core import Rng

pytestmark = pytest.mark.gpu


def close(got, want, what):
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6, err_msg=what)
    return float(np.mean(got == want))


def test_som_and_kmeans_small_vs_reference(golden):
    pts, hi0, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    model = esom.LandmarkModel.create(hi0, lo)
    rng = Rng(2)
    for t in range(5):
        model = model.with_hi(esom.som_tick(esom.Dataset.from_points(pts), model,
                                            esom.SomConfig(sigma=0.8, alpha=0.2, batch_size=64), rng))
        close(model.hi, golden["small_som_his"][t], f"som tick {t}")
    model = esom.LandmarkModel.create(hi0, lo)
    rng = Rng(3)
    for t in range(5):
        model = model.with_hi(esom.kmeans_tick(esom.Dataset.from_points(pts), model,
                                               esom.KmeansConfig(alpha_km=0.3, batch_size=64), rng))
        close(model.hi, golden["small_km_his"][t], f"kmeans tick {t}")


def test_c3_online_ticks_vs_reference(golden):
    pts, hi, lo = c2_inputs()
    model = esom.LandmarkModel.create(hi, lo)
    X = torch.from_numpy(pts).cuda()
    got = esom.som_tick(X, model, esom.SomConfig(sigma=1.0, alpha=0.1), Rng(7)).cpu().numpy()
    assert close(got, golden["c3_som_hi"], "c3 som") > 0.9
    got = esom.kmeans_tick(X, model, esom.KmeansConfig(), Rng(8)).cpu().numpy()
    assert close(got, golden["c3_km_hi"], "c3 kmeans") > 0.99


def test_som_properties(golden):
    pts, hi0, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    ds = esom.Dataset.from_points(pts)
    model = esom.LandmarkModel.create(hi0, lo)
    out = esom.som_tick(ds, model, esom.SomConfig(sigma=1.0, alpha=0.0), Rng(3))
    assert np.array_equal(out, model.hi)                       # tests:test_som.py:40-44
    before = model.lo.copy()
    esom.som_tick(ds, model, esom.SomConfig(), Rng(6))
    assert np.array_equal(model.lo, before)                    # tests:test_som.py:105-109
    one = esom.LandmarkModel.create(np.zeros((1, 5), np.float32), np.zeros((1, 2), np.float32))
    s = int(Rng(9).integers(0, 500, size=1)[0])
    out = esom.som_tick(ds, one, esom.SomConfig(sigma=1.0, alpha=1.0, batch_size=1), Rng(9))
    np.testing.assert_array_equal(out[0], pts[s])              # tests:test_som.py:46-54
    big = esom.som_tick(ds, model, esom.SomConfig(sigma=2.0, alpha=0.3, batch_size=1), Rng(8))
    small = esom.som_tick(ds, model, esom.SomConfig(sigma=0.5, alpha=0.3, batch_size=1), Rng(8))
    assert np.all(np.linalg.norm(small - model.hi, axis=1) <= np.linalg.norm(big - model.hi, axis=1) + 1e-12)


def test_quantization_error(golden):
    pts, hi0 = golden["small_points"], golden["small_hi0"]
    qe = esom.quantization_error(esom.Dataset.from_points(pts), hi0)
    assert qe == pytest.approx(float(golden["small_qe"][0]), rel=1e-6)


def test_som_efficacy_c06():
    # tests:test_acceptance.py:203-221 on the device trainer
    ds = esom.Dataset.from_points(datagen.extruded_s(10_000, seed=5))
    rng = Rng(2)
    hi = ds.points[rng.choice_distinct(ds.n, 256)]
    model = esom.LandmarkModel.create(hi, datagen.lattice(16, 16))
    before = esom.quantization_error(ds, model.hi)
    for t in range(50):
        cfg = esom.SomConfig(sigma=1.5 + (0.2 - 1.5) * t / 49, alpha=0.1)
        model = model.with_hi(esom.som_tick(ds, model, cfg, rng))
    assert esom.quantization_error(ds, model.hi) <= 0.7 * before


def test_batch_som_vs_oracle(golden):
    pts, hi0, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    model = esom.LandmarkModel.create(hi0, lo)
    for mode, m in (("mean_field", 0), ("kohonen", 1)):
        got = batch_som_step(pts, model, BatchSomConfig(sigma=0.9, alpha=0.3, mode=mode))
        want = oracle.batch_som_step(pts, hi0, lo, 0.9, 0.3, m)
        close(got, want, mode)
    pts2, hi2, lo2 = c2_inputs()
    sub = pts2[: 1 << 17]
    got = batch_som_step(torch.from_numpy(sub).cuda(), esom.LandmarkModel.create(hi2, lo2),
                         BatchSomConfig(sigma=1.0, alpha=0.1)).cpu().numpy()
    want = oracle.batch_som_step(sub, hi2, lo2, 1.0, 0.1)
    close(got, want, "c3 batch")


def test_batch_som_b1_equals_online(golden):
    pts, hi0, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    model = esom.LandmarkModel.create(hi0, lo)
    for s in (3, 77, 401):
        batch = batch_som_step(pts[s:s + 1], model, BatchSomConfig(sigma=0.8, alpha=0.4))
        online = oracle.som_tick(pts, hi0, lo, np.array([s]), 0.8, 0.4)
        np.testing.assert_allclose(batch, online, rtol=1e-6, atol=1e-7)


def test_frame_loop_trains_and_embeds():
    pts, hi, lo = c2_inputs()
    X = torch.from_numpy(pts).cuda()
    loop = FrameLoop(X, hi, lo, 16, BatchSomConfig(sigma=0.3, alpha=0.5))
    qes = []
    for _ in range(5):
        loop.frame()
        qes.append(float(loop.qe.item()) / pts.shape[0])
    assert qes[-1] < qes[0]
    assert torch.isfinite(loop.xy).all()
    # the frame's embedding equals a standalone embed under the same landmarks
    hi_now = loop.model.hi.clone()
    xy_loop = loop.frame().clone()
    xy_ref = esom.embed(X, esom.LandmarkModel.create(hi_now.cpu().numpy(), lo), esom.EmbedParams(k=16))
    assert torch.equal(xy_loop, xy_ref)


@pytest.mark.parametrize("g,d", [(4, 4), (64, 32), (256, 32), (1024, 32), (300, 48), (256, 64), (512, 100)])
@pytest.mark.parametrize("variant", ["auto", "ESOM_TICK_REG", "ESOM_TICK_SMEM", "ESOM_TICK_GLOBAL"])
def test_online_tick_kernels_vs_oracle(g, d, variant, monkeypatch):
    """Every online-tick kernel (row-per-thread / register / shared-memory
    cluster / global) against the C restatement of som_tick / kmeans_tick."""
    if variant != "auto":
        monkeypatch.setenv(variant, "1")
    pts = datagen.gaussians(8, 20000, d, seed=3)[0].astype(np.float32)
    gen = np.random.default_rng(g * 131 + d)
    hi = pts[gen.choice(len(pts), g, replace=False)].copy()
    lo = gen.uniform(0, 6, size=(g, 2)).astype(np.float32)
    model = esom.LandmarkModel.create(hi, lo)
    X = torch.from_numpy(pts).cuda()
    cfg = esom.SomConfig(sigma=0.9, alpha=0.3, batch_size=200)
    got = esom.som_tick(X, model, cfg, Rng(5)).cpu().numpy()
    want = oracle.som_tick(pts, hi, lo, Rng(5).integers(0, len(pts), size=200), 0.9, 0.3)
    assert close(got, want, f"som g={g} d={d} {variant}") > 0.5
    kcfg = esom.KmeansConfig(alpha_km=0.2, batch_size=200)
    got = esom.kmeans_tick(X, model, kcfg, Rng(6)).cpu().numpy()
    want = oracle.kmeans_tick(pts, hi, Rng(6).integers(0, len(pts), size=200), 0.2)
    assert close(got, want, f"kmeans g={g} d={d} {variant}") > 0.9


def test_sharded_online_ticks_single_rank_equal_plain():
    from paper_2201_00701_b200.sharded import kmeans_tick_sharded, som_tick_sharded

    pts, hi, lo = c2_inputs()
    model = esom.LandmarkModel.create(hi, lo)
    X = torch.from_numpy(pts).cuda()
    a = som_tick_sharded(X, 0, X.shape[0], model, esom.SomConfig(), Rng(4)).cpu().numpy()
    b = esom.som_tick(X, model, esom.SomConfig(), Rng(4)).cpu().numpy()
    assert np.array_equal(a, b)
    a = kmeans_tick_sharded(X, 0, X.shape[0], model, esom.KmeansConfig(), Rng(5)).cpu().numpy()
    b = esom.kmeans_tick(X, model, esom.KmeansConfig(), Rng(5)).cpu().numpy()
    assert np.array_equal(a, b)


def test_frame_loop_cuda_graph_replay_equals_eager():
    """bench.py times one CUDA-graph launch per frame: replaying the captured
    frame (fused embed + BMU statistics + update + re-preparation) must give
    the landmarks and positions of eager frames."""
    pts, hi, lo = c2_inputs()
    X = torch.from_numpy(pts[:200_000]).cuda()
    a = FrameLoop(X, hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
    b = FrameLoop(X, hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
    for _ in range(3):
        a.frame()
    b.capture()  # one eager frame, then one recorded (not executed) frame
    for _ in range(2):
        b.frame()
    torch.cuda.synchronize()
    # exact integer statistics: replay and eager frames are bit-identical
    assert torch.equal(a.model.hi, b.model.hi)
    assert torch.equal(a.xy, b.xy)


@pytest.mark.parametrize("shape", [(16, 16, 200_000), (32, 32, 300_000)])
def test_frame_loop_training_is_deterministic(shape):
    """Two loops over the same points -- one in natural row order, one over a
    row permutation, the C3 (shared-memory table) and C4 (BMU-sorted segment
    sums) statistics paths -- reach bit-identical landmarks after 5 frames."""
    rows, cols, n = shape
    pts = datagen.gaussians(16, n, 32, seed=1)[0].astype(np.float32)
    hi, lo = datagen.som_model(pts, rows, cols, seed=2)
    perm = np.random.default_rng(5).permutation(n)
    a = FrameLoop(torch.from_numpy(pts).cuda(), hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
    b = FrameLoop(torch.from_numpy(pts[perm]).cuda(), hi, lo, 16, BatchSomConfig(sigma=1.0, alpha=0.05))
    assert a.fx == b.fx
    for _ in range(5):
        a.frame()
        b.frame()
    assert torch.equal(a.model.hi, b.model.hi)


def test_batch_som_fixed_point_vs_oracle(golden):
    """The device statistics equal the oracle's integer restatement exactly."""
    from paper_2201_00701_b200.batch_som import accumulate, dataset_fx_bits, new_acc

    pts, hi, lo = c2_inputs()
    X = torch.from_numpy(pts[: 1 << 17]).cuda()
    H = torch.from_numpy(hi).cuda()
    fx = dataset_fx_bits(X)
    acc = new_acc(*hi.shape, X.device)
    accumulate(X, H, acc, fx)
    S, C = oracle.batch_som_accumulate_fx(pts[: 1 << 17], hi, fx)
    got = acc.cpu().numpy()
    gd = hi.size
    assert np.array_equal(got[:gd].reshape(hi.shape), S) and np.array_equal(got[gd:], C)


def test_frame_loop_capture_keeps_the_census_decision():
    """The far-point census of the eager warm-up frames decides the visiting
    order (BMU order for far-heavy, i.e. trained, models); capturing the frame
    graph afterwards must keep that decision (a second census on the zeroed
    counter used to switch it off for every captured frame)."""
    pts, hi, lo = c2_inputs()
    X = torch.from_numpy(pts[:200_000]).cuda()
    model = esom.LandmarkModel.create(hi, lo)
    rng = Rng(3)

    class _D:
        points = X

    for _ in range(40):  # the interactive steady state: a trained SOM, far-point heavy
        model = esom.LandmarkModel.create(esom.som_tick(_D, model, esom.SomConfig(), rng).cpu().numpy(), lo)
    eager = FrameLoop(X, model.hi, lo, 16, train=False)
    for _ in range(3):
        eager.frame()
    assert eager.bmu_order  # (the census found the far-heavy regime)
    cap = FrameLoop(X, model.hi, lo, 16, train=False)
    for _ in range(3):
        cap.frame()
    cap.capture()
    assert cap.bmu_order
    cap.frame()
    torch.cuda.synchronize()
    assert torch.equal(cap.xy, eager.xy)
    fresh = FrameLoop(X, model.hi, lo, 16, train=False)
    fresh.capture()  # census from capture's own eager frame
    assert fresh.bmu_order
