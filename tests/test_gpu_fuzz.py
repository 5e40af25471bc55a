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


def _train_shapes():
    gen = np.random.default_rng(777)
    out = []
    for _ in range(16):
        d = int(gen.choice([1, 3, 8, 17, 32, 33, 64, 65, 100]))
        g = int(gen.choice([4, 7, 36, 64, 200, 256, 257, 700, 1024, 2000]))
        B = int(gen.choice([1, 2, 63, 64, 65, 200, 256, 300]))
        out.append((d, g, B, int(gen.integers(1 << 30))))
    return out


@pytest.mark.parametrize("d,g,B,seed", _train_shapes())
def test_fuzz_trainers(d, g, B, seed):
    """Online SOM / k-means ticks (every on-chip / global kernel variant the
    shape selects) and the batch-SOM step against the C restatements."""
    from paper_2201_00701_b200.core import Rng

    gen = np.random.default_rng(seed)
    n = 5000
    centers = gen.uniform(0, 10, size=(5, d))
    pts = (centers[gen.integers(0, 5, n)] + gen.normal(0, 0.5, size=(n, d))).astype(np.float32)
    hi = pts[gen.choice(n, g, replace=g > n)].copy()
    lo = gen.uniform(0, 6, size=(g, 2)).astype(np.float32)
    model = esom.LandmarkModel.create(hi, lo)
    X = torch.from_numpy(pts).cuda()
    got = esom.som_tick(X, model, esom.SomConfig(sigma=0.9, alpha=0.3, batch_size=B), Rng(seed)).cpu().numpy()
    want = oracle.som_tick(pts, hi, lo, Rng(seed).integers(0, n, size=B), 0.9, 0.3)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5, err_msg=f"som {d} {g} {B}")
    got = esom.kmeans_tick(X, model, esom.KmeansConfig(alpha_km=0.2, batch_size=B), Rng(seed + 1)).cpu().numpy()
    want = oracle.kmeans_tick(pts, hi, Rng(seed + 1).integers(0, n, size=B), 0.2)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5, err_msg=f"kmeans {d} {g} {B}")
    got = esom.batch_som_step(X, model, esom.BatchSomConfig(sigma=1.1, alpha=0.2)).cpu().numpy()
    want = oracle.batch_som_step(pts, hi, lo, 1.1, 0.2)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5, err_msg=f"batch {d} {g}")


def _api_shapes():
    gen = np.random.default_rng(4242)
    out = []
    for _ in range(14):
        d = int(gen.choice([1, 2, 7, 32, 50, 200]))
        g = int(gen.choice([1, 2, 5, 65, 130, 300, 1100]))
        k = int(gen.choice([1, 2, 3, 17, 65, 100]))
        k = max(1, min(k, g))
        n = int(gen.choice([0, 1, 3, 999, 4097]))
        out.append((n, d, g, k, int(gen.integers(1 << 30))))
    return out


@pytest.mark.parametrize("n,d,g,k,seed", _api_shapes())
def test_fuzz_api_paths(n, d, g, k, seed):
    """knn / knn_bitonic / project_neighbors / chunked embed on odd shapes
    (k > 64 sort path, k < 3, g = 1, n = 0, float64 and strided inputs)."""
    gen = np.random.default_rng(seed)
    pts64 = gen.normal(0, 3, size=(n, d))
    pts = pts64.astype(np.float32)
    hi = gen.normal(0, 3, size=(g, d)).astype(np.float32)
    lo = gen.uniform(0, 5, size=(g, 2)).astype(np.float32)
    nb = esom.knn(pts64, hi, k, backend="base")  # float64 in: coerced like the reference
    wi, wd = oracle.knn(pts, hi, k) if n else (np.zeros((0, k), np.int32), np.zeros((0, k), np.float32))
    assert np.array_equal(nb.indices, wi) and np.array_equal(nb.sqdists, wd)
    if k in (4, 8, 16, 32, 64):
        nb2 = esom.knn_bitonic(np.asfortranarray(pts), hi, k)  # strided input
        assert np.array_equal(nb2.indices, wi) and np.array_equal(nb2.sqdists, wd)
    if k >= 3 and n:
        model = esom.LandmarkModel.create(hi, lo)
        xy = esom.project_neighbors(pts, model, nb)
        ref = oracle.project(pts, hi, lo, wi, oracle.scores(wd))
        ext = max(float(np.ptp(lo, axis=0).max()), 1e-30)
        assert np.abs(xy - ref).max() <= 1e-4 * ext
        full = esom.embed(pts, model, esom.EmbedParams(k=k), backend="base")
        chunked = esom.embed(pts, model, esom.EmbedParams(k=k), backend="base", chunk_size=max(1, n // 3))
        assert np.array_equal(full, chunked)  # chunk invariance (ref: tests:test_projection.py:217-223)


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_formats_and_landmark_ops(seed):
    """FCS images (random n, d, byte order, header/TEXT offsets), transforms,
    colours, frame records, graph + layout + fit_hi on random inputs vs the
    numpy restatements (oracle/formats.py)."""

    from oracle import formats as F
    from paper_2201_00701_b200.engine import DeviceSession
    from paper_2201_00701_b200.io import TransformSpec, apply_transform, parse_fcs

    gen = np.random.default_rng(9000 + seed)
    n, d = int(gen.integers(1, 3000)), int(gen.integers(1, 40))
    pts = (gen.normal(0, 1, size=(n, d)) * gen.uniform(0.1, 100, size=d)).astype(np.float32)
    big = bool(gen.integers(2))
    text_offsets = bool(gen.integers(2))
    kws = [("$PAR", str(d)), ("$TOT", str(n)), ("$DATATYPE", "F"), ("$BYTEORD", "4,3,2,1" if big else "1,2,3,4"),
           ("$MODE", "L")] + [(f"$P{i + 1}B", "32") for i in range(d)] + [(f"$P{i + 1}N", f"c/{i}") for i in range(d)]
    pad = int(gen.integers(0, 7))  # unaligned DATA offsets
    def text(b0, b1):
        extra = [("$BEGINDATA", f"{b0:010d}"), ("$ENDDATA", f"{b1:010d}")] if text_offsets else []
        return b"/" + b"".join(k.encode().replace(b"/", b"//") + b"/" + v.encode().replace(b"/", b"//") + b"/"
                               for k, v in kws + extra)
    t = text(0, 0)
    d0 = 58 + len(t) + pad
    d1 = d0 + 4 * n * d - 1
    t = text(d0, d1)
    hdr = (b"FCS3.1    " + b"".join(f"{v:>8d}".encode() for v in
                                      (58, 58 + len(t) - 1, 0 if text_offsets else d0, 0 if text_offsets else d1, 0, 0)))
    raw = hdr + t + b"\0" * pad + pts.astype(">f4" if big else "<f4").tobytes()
    ds = parse_fcs(raw)
    assert np.array_equal(ds.points.cpu().numpy(), pts)
    assert ds.dim_names == tuple(f"c/{i}" for i in range(d))
    spec = tuple(gen.choice(["none", "minmax", "zscore"]) for _ in range(d))
    out = apply_transform(ds, TransformSpec(entries=spec)).points.cpu().numpy()
    st = ds.dim_stats
    want = F.apply_transform(pts, spec, (st.min, st.max, st.mean, st.sd))
    assert np.array_equal(out, want)  # bit-exact given the statistics
    sess = DeviceSession(pts)
    c = int(gen.integers(d))
    assert np.array_equal(sess.colors(c).cpu().numpy(), F.color_channel(pts, pts.min(0), pts.max(0), c))
    xy = gen.normal(0, 5, size=(n, 2)).astype(np.float32)
    sess.positions.copy_(torch.from_numpy(xy))
    fid = int(gen.integers(0, 2**32))
    assert bytes(sess.frame_record(fid, c)) == F.frame_points_record(fid, xy, sess.colors(c).cpu().numpy())
    # landmark-side ops
    g = int(gen.integers(5, 300))
    hi = gen.normal(0, 2, size=(g, d)).astype(np.float32)
    lo = gen.uniform(0, 6, size=(g, 2)).astype(np.float32)
    kg = int(gen.integers(1, min(8, g - 1) + 1))
    e = esom.build_knn_graph(hi, kg)
    from paper_2201_00701_b200.graphmodel import symmetrize_neighbors
    wi, wd = oracle.knn(hi, hi, kg + 1)
    e2 = symmetrize_neighbors(wi, wd, kg)
    assert np.array_equal(e.pairs, e2.pairs) and np.array_equal(e.rest, e2.rest)
    lay = esom.LayoutState(velocities=gen.normal(0, 0.1, size=(g, 2)))
    pinned = sorted(set(gen.integers(0, g, size=3).tolist()))
    new_lo, vel = esom.layout_tick(lo, e, lay, pinned)
    wlo, wvel = F.layout_tick(lo, e.pairs, e.rest, lay.velocities, lay.stiffness, lay.repulsion, 1e-3, lay.damping,
                              lay.dt, pinned)
    np.testing.assert_allclose(vel, wvel, rtol=1e-9, atol=1e-12)
    assert np.max(np.abs(new_lo - wlo)) <= 1e-5
    model = esom.LandmarkModel.create(hi, lo)
    p = gen.uniform(-1, 7, size=2)
    np.testing.assert_allclose(esom.fit_hi_for_new_landmark(p, model), F.fit_hi_for_new_landmark(p, hi, lo),
                               rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("n,d,g,k", [((1 << 20) + 77, 32, 300, 16), ((1 << 18) + 123, 40, 600, 20),
                                     ((1 << 18) + 1, 130, 257, 32)])
def test_chunk_boundaries_vs_scan(n, d, g, k, monkeypatch):
    """Screens that work in chunks (split tc2: 2^20 points; GEMM screen: <= 2^18)
    with a ragged last chunk, bit-exact against the CUDA-core scan."""
    gen = np.random.default_rng(n + d)
    centers = gen.uniform(0, 10, size=(8, d)).astype(np.float32)
    X = torch.from_numpy(centers[gen.integers(0, 8, n)] + gen.normal(0, 0.5, size=(n, d)).astype(np.float32)).cuda()
    H = torch.from_numpy(centers[gen.integers(0, 8, g)] + gen.normal(0, 0.7, size=(g, d)).astype(np.float32)).cuda()
    a = esom.knn_base(X, H, k)
    monkeypatch.setenv("ESOM_TC", "0")
    b = esom.knn_base(X, H, k)
    assert torch.equal(a.indices, b.indices) and torch.equal(a.sqdists, b.sqdists)


@pytest.mark.parametrize("n,d,g,k,seed", [(3000, 5, 40, 8, 1), (50000, 32, 256, 16, 2), (20000, 32, 1024, 16, 3),
                                          (8000, 48, 300, 32, 4), (4097, 2, 9, 4, 5), (12000, 70, 100, 16, 6)])
def test_fuzz_frame_loop(n, d, g, k, seed):
    """Batch-SOM FrameLoop (fused embed + statistics via the shared-memory or
    sorted-segment kernel + update + re-preparation) for two frames vs the C
    restatements: positions of each frame under that frame's model, hi after."""
    from paper_2201_00701_b200.batch_som import BatchSomConfig, FrameLoop

    gen = np.random.default_rng(seed)
    centers = gen.uniform(0, 10, size=(6, d))
    pts = (centers[gen.integers(0, 6, n)] + gen.normal(0, 0.5, size=(n, d))).astype(np.float32)
    hi = pts[gen.choice(n, g, replace=False)].copy()
    lo = gen.uniform(0, 6, size=(g, 2)).astype(np.float32)
    loop = FrameLoop(torch.from_numpy(pts).cuda(), hi, lo, k, BatchSomConfig(sigma=1.0, alpha=0.1))
    ext = float(np.ptp(lo, axis=0).max())
    h = hi
    for _ in range(2):
        xy = loop.frame().cpu().numpy()
        ref = oracle.embed(pts, h, lo, k, threads=oracle.host_cores())
        assert np.abs(xy - ref).max() <= 1e-4 * ext
        h = oracle.batch_som_step(pts, h, lo, 1.0, 0.1)
        np.testing.assert_allclose(loop.model.hi.cpu().numpy(), h, rtol=1e-5, atol=1e-5)
