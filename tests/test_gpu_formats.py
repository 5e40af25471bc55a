"""Device kernels of the rows either side of the embed path
against the reference-generated fixtures (tests/golden/make_golden_frames.py)
and the numpy oracle (oracle/formats.py):

* colours (esom_color_channel) and FramePoints records (esom_frame_points_pack)
  bit-exact, including every record length mod 16 and the mapped-host write;
* FCS DATA decode bit-exact (both byte orders, FCS3.1 offsets), errors as the
  reference; statistics min/max exact, mean/sd to 1e-12 relative;
* transforms bit-exact given the reference's statistics, <= 1 f32 ulp with
  the device statistics;
* FrameEngine (device-resident Engine.tick) vs the reference Engine's frames.
"""
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import formats as F
import paper_2201_00701_b200 as esom
from paper_2201_00701_b200 import datagen
from paper_2201_00701_b200.core import InputError, ParseError
from paper_2201_00701_b200.engine import DeviceSession, FrameEngine
from paper_2201_00701_b200.io import (DeviceDataset, DimStats, TransformSpec, apply_transform, compute_dim_stats,
                                      parse_fcs)
from paper_2201_00701_b200.protocol import FrameBuffer, encode_frame_points, pack_frame_points

pytestmark = pytest.mark.gpu
META = json.loads((GOLDEN / "golden_frames.json").read_text())


@pytest.fixture(scope="module")
def gf():
    return np.load(GOLDEN / "golden_frames.npz")


def test_color_channel_bit_exact(gf):
    for key in ("col", "col2"):
        sess = DeviceSession(gf[f"{key}_points"])
        m64 = gf[f"{key}_points"].astype(np.float64)
        assert np.array_equal(sess.col_min, m64.min(axis=0)) and np.array_equal(sess.col_max, m64.max(axis=0))
        for c in range(gf[f"{key}_points"].shape[1]):
            assert np.array_equal(sess.colors(c).cpu().numpy(), gf[f"{key}_colors"][c]), (key, c)
    with pytest.raises(esom.ParameterError, match="out of range"):
        sess.colors(99)


def test_frame_record_bit_exact(gf):
    for i, r in enumerate(META["records"]):
        got = encode_frame_points(r["frame_id"], torch.from_numpy(gf[f"rec{i}_pos"]).cuda(),
                                  torch.from_numpy(gf[f"rec{i}_col"]).cuda())
        assert got == gf[f"rec{i}_bytes"].tobytes(), r


def test_frame_record_all_tails_and_staging():
    rng = np.random.default_rng(5)
    buf = FrameBuffer(13 + 9 * 300)
    assert buf.dev_ptr is not None  # pinned host memory is mapped (UVA): the kernel writes it directly
    staged = FrameBuffer(13 + 9 * 300)
    staged.staging, staged.dev_ptr = torch.empty(staged.capacity, dtype=torch.uint8, device="cuda"), None
    for n in list(range(0, 40)) + [255, 256, 257, 300]:
        pos = rng.normal(size=(n, 2)).astype(np.float32)
        col = rng.integers(0, 256, n).astype(np.uint8)
        want = F.frame_points_record(n * 7 + 3, pos, col)
        for b in (buf, staged):
            b.host.fill_(0xAB)
            nb = pack_frame_points(torch.from_numpy(pos).cuda(), torch.from_numpy(col).cuda(), n * 7 + 3, b)
            b.event.synchronize()
            assert bytes(b.host[:nb].numpy()) == want, n
            if nb < b.capacity:
                assert int(b.host[nb]) == 0xAB  # nothing written past the record


def test_parse_fcs_bit_exact_and_errors(gf):
    checked = 0
    for ent in META["fcs"]:
        raw = gf[f"fcs_{ent['name']}_raw"].tobytes()
        if "error" in ent:
            cls = InputError if ent["error"] == "InputError" else ParseError
            with pytest.raises(cls) as ei:
                parse_fcs(raw)
            assert str(ei.value) == ent["message"], ent["name"]
            continue
        ds = parse_fcs(raw)
        name = ent["name"]
        assert ds.dim_names == tuple(ent["names"])
        assert np.array_equal(ds.points.cpu().numpy(), gf[f"fcs_{name}_points"]), name
        st = ds.dim_stats
        assert np.array_equal(st.min, gf[f"fcs_{name}_min"]) and np.array_equal(st.max, gf[f"fcs_{name}_max"])
        np.testing.assert_allclose(st.mean, gf[f"fcs_{name}_mean"], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(st.sd, gf[f"fcs_{name}_sd"], rtol=1e-12, atol=1e-300)
        checked += 1
    assert checked >= 20


def test_dim_stats_large_vs_numpy():
    pts = datagen.gaussians(16, 300_000, 32, seed=9)[0].astype(np.float32) * 100
    st = compute_dim_stats(torch.from_numpy(pts).cuda())
    mn, mx, mean, sd = F.dim_stats(pts)
    assert np.array_equal(st.min, mn) and np.array_equal(st.max, mx)
    np.testing.assert_allclose(st.mean, mean, rtol=1e-12)
    np.testing.assert_allclose(st.sd, sd, rtol=1e-12)


def test_transforms_bit_exact_given_stats(gf):
    for ent in META["transforms"]:
        name = ent["name"]
        entries = tuple(e if isinstance(e, str) else tuple(e) for e in ent["entries"])
        s = gf[f"xf_{name}_stats_in"]
        ds = DeviceDataset(points=torch.from_numpy(gf[f"xf_{name}_in"]).cuda(),
                           dim_names=tuple(f"dim{i}" for i in range(s.shape[1])),
                           dim_stats=DimStats(min=s[0], max=s[1], mean=s[2], sd=s[3]))
        out = apply_transform(ds, TransformSpec(entries=entries))
        assert np.array_equal(out.points.cpu().numpy(), gf[f"xf_{name}_out"]), name
        # end to end with the device statistics: within one f32 ulp
        out2 = apply_transform(DeviceDataset.from_points(gf[f"xf_{name}_in"]), TransformSpec(entries=entries))
        got, want = out2.points.cpu().numpy(), gf[f"xf_{name}_out"]
        assert np.all(np.abs(got - want) <= np.spacing(np.abs(want).astype(np.float32)) + 1e-30), name
    with pytest.raises(esom.ParameterError):
        apply_transform(DeviceDataset.from_points(np.ones((5, 3), np.float32)), TransformSpec.uniform("zscore", 2))
    with pytest.raises(InputError, match="non-finite"):
        DeviceDataset.from_points(np.array([[1.0, np.inf]], np.float32))


def test_frame_engine_vs_reference_engine(gf):
    eng = FrameEngine(gf["col_points"], seed=META["engine"]["seed"], k=16, grid=tuple(META["engine"]["grid"]))
    assert np.array_equal(eng.model.hi, gf["eng_hi0"])
    assert eng.embed_params.k == META["engine"]["k_eff"]
    ext = float(np.ptp(gf["eng_lo"], axis=0).max())
    for t, tk in enumerate(META["engine"]["ticks"]):
        fr = eng.tick()
        assert fr.frame_id == tk["frame_id"]
        np.testing.assert_allclose(eng.model.hi, gf[f"eng_hi{t + 1}"], rtol=1e-5, atol=1e-6)
        err = np.abs(fr.positions.cpu().numpy() - gf[f"eng_pos{t}"]).max()
        assert err <= 1e-4 * ext, (t, err)
        rec = bytes(eng.frame_record())
        assert len(rec) == tk["len"]
        assert rec == F.frame_points_record(tk["frame_id"], fr.positions.cpu().numpy(), gf["eng_colors"])
    assert np.array_equal(fr.colors.cpu().numpy(), gf["eng_colors"])


def test_frame_engine_replay_is_deterministic():
    pts = datagen.extruded_s(5000, seed=4)
    recs = []
    for _ in range(2):
        eng = FrameEngine(pts, seed=1234, k=16, grid=(8, 8))
        recs.append([bytes(eng.tick() and eng.frame_record()) for _ in range(5)])
    assert recs[0] == recs[1]
    other = FrameEngine(pts, seed=1235, k=16, grid=(8, 8))
    assert bytes(other.tick() and other.frame_record()) != recs[0][0]


def test_landmark_graph_and_layout_vs_reference(gf):
    e = esom.build_knn_graph(gf["eng_hi0"], 3)
    assert np.array_equal(e.pairs, gf["graph_pairs"]) and np.array_equal(e.rest, gf["graph_rest"])
    hi4096 = datagen.gaussians(16, 4096, 32, seed=7)[0].astype(np.float32)
    e2 = esom.build_knn_graph(torch.from_numpy(hi4096).cuda(), 8)
    assert np.array_equal(e2.pairs, gf["graph4096_pairs"]) and np.array_equal(e2.rest, gf["graph4096_rest"])
    lay = META["layout"]
    st = esom.LayoutState(velocities=gf["layout_vel0"], stiffness=lay["stiffness"], repulsion=lay["repulsion"],
                          damping=lay["damping"], dt=lay["dt"])
    f = esom.net_forces(gf["layout_lo0"], e, st)
    np.testing.assert_allclose(f, gf["layout_forces"], rtol=1e-12, atol=1e-12)
    lo1, v1 = esom.layout_tick(gf["layout_lo0"], e, st, pinned_rows=lay["pinned"])
    np.testing.assert_allclose(v1, gf["layout_vel1"], rtol=1e-12, atol=1e-13)
    assert np.max(np.abs(lo1 - gf["layout_lo1"])) <= 1e-6
    assert np.array_equal(lo1[lay["pinned"]], gf["layout_lo0"][lay["pinned"]])
    assert np.all(v1[lay["pinned"]] == 0)
    # g = 4096 layout (where the device pays off) vs the numpy restatement
    lo4 = datagen.extruded_s(4096, seed=2)[:, :2].astype(np.float32) * 10
    st4 = esom.LayoutState.for_count(4096)
    lo4b, v4 = esom.layout_tick(lo4, e2, st4)
    want_lo, want_v = F.layout_tick(lo4, e2.pairs, e2.rest, st4.velocities, st4.stiffness, st4.repulsion, 1e-3,
                                    st4.damping, st4.dt)
    np.testing.assert_allclose(v4, want_v, rtol=1e-9, atol=1e-12)
    assert np.max(np.abs(lo4b - want_lo)) <= 1e-5


def test_fit_hi_for_new_landmark_vs_reference(gf):
    model = esom.LandmarkModel.create(gf["eng_hi0"], gf["eng_lo"])
    for p, want in zip(gf["fit_pos"], gf["fit_hi"]):
        np.testing.assert_allclose(esom.fit_hi_for_new_landmark(p, model), want, rtol=1e-6)
    assert np.array_equal(esom.fit_hi_for_new_landmark((0.0, 0.0), model), gf["eng_hi0"][0])  # exact hit
    with pytest.raises(InputError, match="2-vector"):
        esom.fit_hi_for_new_landmark((1.0, 2.0, 3.0), model)


def _fake_reference_engine(points, seed, grid, k, chunk_size=131072):
    """The attributes of embedview.engine.Engine that gpu_tick touches, so the
    installed tick runs here without the reference (ref: engine.py:109-236)."""
    import dataclasses
    import sys
    import types

    from paper_2201_00701_b200 import graphmodel as G
    from paper_2201_00701_b200.core import EmbedParams, Rng
    from paper_2201_00701_b200.engine import _nearest_pow2_k, init_model

    mod = types.ModuleType("fake_embedview_engine")
    mod.MODE_SOM, mod.MODE_GRAPH = "som", "graph"
    mod.FramePacket = dataclasses.make_dataclass(
        "FramePacket", ["frame_id", "positions", "landmarks_lo", "landmark_ids", "edges", "colors"])
    mod.EdgeSet, mod.graphmodel, mod.replace = G.EdgeSet, G, dataclasses.replace
    sys.modules[mod.__name__] = mod
    Eng = type("Engine", (), {"__module__": mod.__name__, "tick": esom.engine.gpu_tick,
                              "apply_command": lambda self, c: None})
    e = Eng()
    rng = Rng(seed)
    ds = esom.Dataset.from_points(points)
    model = init_model(ds.points, rng, grid)
    e.state = types.SimpleNamespace(dataset=ds, model=model, mode="som", som_cfg=esom.SomConfig(),
                                    km_cfg=esom.KmeansConfig(), rng=rng, training_paused=False, chunk_cursor=0,
                                    frame_id=0, color_dim=0, edges=G.EdgeSet.empty(),
                                    embed_params=EmbedParams(k=_nearest_pow2_k(k, model.g)))
    e._queue, e._errors, e._colors, e.chunk_size, e.backend = [], [], None, chunk_size, "bitonic"
    e._positions = np.zeros((ds.n, 2), np.float32)
    return e


def test_installed_gpu_tick_vs_reference_engine(gf):
    e = _fake_reference_engine(gf["col_points"], META["engine"]["seed"], tuple(META["engine"]["grid"]), 16)
    ext = float(np.ptp(gf["eng_lo"], axis=0).max())
    for t, tk in enumerate(META["engine"]["ticks"]):
        p = e.tick()
        assert p.frame_id == tk["frame_id"] and isinstance(p.positions, np.ndarray)
        np.testing.assert_allclose(e.state.model.hi, gf[f"eng_hi{t + 1}"], rtol=1e-5, atol=1e-6)
        assert np.abs(p.positions - gf[f"eng_pos{t}"]).max() <= 1e-4 * ext
        assert np.array_equal(p.colors, gf["eng_colors"])


def test_installed_gpu_tick_round_robin_chunks():
    pts = datagen.extruded_s(3000, seed=6)
    full = _fake_reference_engine(pts, 5, (6, 6), 16)
    rr = _fake_reference_engine(pts, 5, (6, 6), 16, chunk_size=1024)
    rr.full_reprojection = False
    full.state.training_paused = rr.state.training_paused = True  # fixed model: chunks converge to the full frame
    want = full.tick().positions
    got = [rr.tick().positions for _ in range(3)]
    assert np.array_equal(got[0][1024:], np.zeros((3000 - 1024, 2), np.float32))
    assert rr.state.chunk_cursor == 0
    assert np.array_equal(got[2], want)


def test_installed_gpu_tick_graph_mode():
    """Graph mode through the installed tick: k-means trainer, k_g-NN graph
    rebuild, device force layout (ref: engine.py:356-375), then the embed."""
    from oracle import oracle as O
    from paper_2201_00701_b200 import graphmodel as G

    pts = datagen.extruded_s(3000, seed=8)
    e = _fake_reference_engine(pts, 3, (6, 6), 16)
    st = e.state
    st.mode, st.k_g = "graph", 3
    st.layout = G.LayoutState.for_count(st.model.g)
    e._edges_dirty, e._ticks_since_rebuild = True, 0

    def rebuild(self=e):
        self.state.edges = G.build_knn_graph(self.state.model.hi, min(self.state.k_g, self.state.model.g - 1))
        self._edges_dirty, self._ticks_since_rebuild = False, 0

    e._rebuild_edges = rebuild
    hi0, lo0 = st.model.hi.copy(), st.model.lo.copy()
    rng_copy = esom.Rng(3)
    esom.engine.init_model(pts, rng_copy, (6, 6))  # advance past the init draw like the engine did
    p = e.tick()
    want_hi = O.kmeans_tick(pts, hi0, rng_copy.integers(0, len(pts), size=256), 0.05)
    np.testing.assert_allclose(st.model.hi, want_hi, rtol=1e-5, atol=1e-6)
    edges = G.build_knn_graph(want_hi, 3)
    lay = G.LayoutState.for_count(len(lo0))
    want_lo, _ = F.layout_tick(lo0, edges.pairs, edges.rest, lay.velocities, lay.stiffness, lay.repulsion, 1e-3,
                               lay.damping, lay.dt)
    assert np.max(np.abs(st.model.lo - want_lo)) <= 1e-5
    assert len(p.edges) == len(edges) and np.all(np.isfinite(p.positions))


def test_session_switches_to_bmu_order_on_trained_models():
    """After a frame in which most points took the far-point path, the session
    visits the projection in nearest-landmark order; per-point results do not
    depend on the visiting order (bit-identical positions)."""
    pts = datagen.gaussians(16, 1 << 16, 32, seed=1)[0].astype(np.float32)
    eng = FrameEngine(pts, seed=7, k=16, grid=(16, 16))
    for _ in range(10):
        eng.tick()
    s = eng.session
    eng.training_paused = True
    first = eng.tick().positions.clone()
    for _ in range(3):  # the census arrives asynchronously: let it land
        torch.cuda.synchronize()
        eng.tick()
    assert s.bmu_order, "trained C3-like model: far-point census should select BMU order"
    assert torch.equal(eng.tick().positions, first)
    fresh = FrameEngine(pts, seed=7, k=16, grid=(16, 16))
    fresh.training_paused = True
    for _ in range(4):
        torch.cuda.synchronize()
        fresh.tick()
    assert not fresh.session.bmu_order  # untrained model: natural order, no sort


def test_frame_engine_pipelined_equals_sequential():
    """The speculative next-tick training on a side stream produces the same
    landmarks, positions and Rng stream as the sequential tick, also across a
    config change (the speculation is rewound)."""
    import dataclasses

    pts = datagen.gaussians(16, 1 << 15, 32, seed=3)[0].astype(np.float32)
    a = FrameEngine(pts, seed=5, k=16, grid=(8, 8), pipelined=True)
    b = FrameEngine(pts, seed=5, k=16, grid=(8, 8), pipelined=False)
    for t in range(6):
        if t == 3:  # change the trainer config between ticks: the speculation must be discarded
            a.som_cfg = b.som_cfg = dataclasses.replace(a.som_cfg, alpha=0.3)
        fa, fb = a.tick(), b.tick()
        assert torch.equal(fa.positions, fb.positions), t
        assert np.array_equal(a.model.hi, b.model.hi), t


def test_installed_gpu_tick_pipelined_equals_sequential():
    """Installed Engine.tick with the speculative next-tick training: commands
    that draw from the session Rng and config changes between ticks rewind it,
    so frames equal the sequential tick's."""
    import dataclasses

    pts = datagen.extruded_s(4000, seed=11)
    engines = [_fake_reference_engine(pts, 21, (6, 6), 16) for _ in range(2)]
    engines[1].pipelined = False
    for e in engines:  # a command that consumes the session Rng (like DuplicateLandmark)
        type(e).apply_command = lambda self, c: self.state.rng.uniform(0.0, 1.0)
    outs = [[], []]
    for t in range(6):
        for i, e in enumerate(engines):
            if t == 2:
                e._queue.append("draw")
            if t == 4:
                e.state.som_cfg = dataclasses.replace(e.state.som_cfg, sigma=0.7)
            p = e.tick()
            outs[i].append((p.positions.copy(), e.state.model.hi.copy()))
    for (pa, ha), (pb, hb) in zip(*outs):
        assert np.array_equal(pa, pb) and np.array_equal(ha, hb)

