"""CPU checks of the rows either side of the embed path:
the numpy oracle (oracle/formats.py) against the reference-generated
fixtures (tests/golden/make_golden_frames.py), and the host-side FCS
HEADER/TEXT parser of the package (same layout, names and error messages as
the reference).  Device kernels are checked in test_gpu_formats.py."""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import formats as F

META = json.loads((GOLDEN / "golden_frames.json").read_text())


@pytest.fixture(scope="module")
def gf():
    return np.load(GOLDEN / "golden_frames.npz")


def test_oracle_color_channel(gf):
    for key in ("col", "col2"):
        pts = gf[f"{key}_points"]
        m64 = pts.astype(np.float64)
        for c in range(pts.shape[1]):
            got = F.color_channel(pts, m64.min(axis=0), m64.max(axis=0), c)
            assert np.array_equal(got, gf[f"{key}_colors"][c]), (key, c)


def test_oracle_frame_record(gf):
    for i, r in enumerate(META["records"]):
        got = F.frame_points_record(r["frame_id"], gf[f"rec{i}_pos"], gf[f"rec{i}_col"])
        assert got == gf[f"rec{i}_bytes"].tobytes()
        assert len(got) == 13 + 9 * r["n"] == r["len"]


def test_fcs_host_parse_and_oracle_decode(gf):
    from paper_2201_00701_b200.core import ParseError
    from paper_2201_00701_b200.io import _fcs_layout

    seen = 0
    for ent in META["fcs"]:
        raw = gf[f"fcs_{ent['name']}_raw"].tobytes()
        if "error" in ent and ent["message"] != "points contains non-finite values":
            with pytest.raises(ParseError) as ei:
                _fcs_layout(raw)
            assert str(ei.value) == ent["message"], ent["name"]
            continue
        n, d, big, d0, names = _fcs_layout(raw)
        pts = F.fcs_decode(raw[d0:d0 + 4 * n * d], n, d, bool(big))
        if "error" in ent:  # non-finite DATA: the Dataset check raises
            assert not np.all(np.isfinite(pts))
            continue
        assert tuple(names) == tuple(ent["names"]), ent["name"]
        assert np.array_equal(pts, gf[f"fcs_{ent['name']}_points"]), ent["name"]
        mn, mx, mean, sd = F.dim_stats(pts)
        assert np.array_equal(mn, gf[f"fcs_{ent['name']}_min"]) and np.array_equal(mx, gf[f"fcs_{ent['name']}_max"])
        assert np.array_equal(mean, gf[f"fcs_{ent['name']}_mean"]) and np.array_equal(sd, gf[f"fcs_{ent['name']}_sd"])
        seen += 1
    assert seen >= 20


def test_oracle_transforms(gf):
    for ent in META["transforms"]:
        name = ent["name"]
        entries = [e if isinstance(e, str) else tuple(e) for e in ent["entries"]]
        got = F.apply_transform(gf[f"xf_{name}_in"], entries)
        assert np.array_equal(got, gf[f"xf_{name}_out"]), name
        st = np.stack(F.dim_stats(got))
        assert np.array_equal(st, gf[f"xf_{name}_stats_out"]), name


def test_oracle_layout_and_fit(gf):
    lay = META["layout"]
    f = F.net_forces(gf["layout_lo0"], gf["graph_pairs"], gf["graph_rest"], lay["stiffness"], lay["repulsion"],
                     lay["eps"])
    np.testing.assert_allclose(f, gf["layout_forces"], rtol=1e-12, atol=1e-12)
    lo1, v1 = F.layout_tick(gf["layout_lo0"], gf["graph_pairs"], gf["graph_rest"], gf["layout_vel0"],
                            lay["stiffness"], lay["repulsion"], lay["eps"], lay["damping"], lay["dt"],
                            lay["pinned"])
    np.testing.assert_allclose(v1, gf["layout_vel1"], rtol=1e-12, atol=1e-13)
    assert np.max(np.abs(lo1 - gf["layout_lo1"])) <= 1e-6
    for p, want in zip(gf["fit_pos"], gf["fit_hi"]):
        got = F.fit_hi_for_new_landmark(p, gf["eng_hi0"], gf["eng_lo"])
        np.testing.assert_allclose(got, want, rtol=1e-6)


def test_engine_init_matches_reference(gf):
    """FrameEngine's model initialisation draws the reference Engine's hi rows."""
    from paper_2201_00701_b200.core import Rng
    from paper_2201_00701_b200.engine import init_model

    m = init_model(gf["col_points"], Rng(META["engine"]["seed"]), tuple(META["engine"]["grid"]))
    assert np.array_equal(m.hi, gf["eng_hi0"]) and np.array_equal(m.lo, gf["eng_lo"])


def test_graph_symmetrize_vs_reference(gf):
    """build_knn_graph's host half on the oracle k-NN rows == the reference's edges."""
    from oracle import oracle
    from paper_2201_00701_b200 import datagen
    from paper_2201_00701_b200.graphmodel import symmetrize_neighbors

    for hi, kg, key in ((gf["eng_hi0"], 3, "graph"),
                        (datagen.gaussians(16, 4096, 32, seed=7)[0].astype(np.float32), 8, "graph4096")):
        idx, sqd = oracle.knn(hi, hi, kg + 1)
        e = symmetrize_neighbors(idx, sqd, kg)
        assert np.array_equal(e.pairs, gf[f"{key}_pairs"]) and np.array_equal(e.rest, gf[f"{key}_rest"]), key


def test_install_reroutes_reference_callers():
    """install() patches the names the reference engine/cli/bench resolve at
    call time -- checked here where the reference exists."""
    import importlib
    import os
    import sys
    from pathlib import Path

    src = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if not (src / "embedview").exists():
        src = Path("/root/reference/pkg/src")
    if not src.exists():
        pytest.skip("reference not present (GPU box)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(src))
    try:
        ev = importlib.import_module("embedview")
        import paper_2201_00701_b200 as esom
        from paper_2201_00701_b200 import engine as E, graphmodel as G, som as S

        esom.install(ev)
        assert importlib.import_module("embedview.engine").Engine.tick is E.gpu_tick
        eng = importlib.import_module("embedview.engine")
        assert eng.embed is esom._faithful_embed and eng.color_channel is E.color_channel
        assert ev.embed is esom._faithful_embed and ev.knn is esom.knn
        assert ev.som.som_tick is S.som_tick and ev.som.fit_hi_for_new_landmark is S.fit_hi_for_new_landmark
        assert ev.graphmodel.layout_tick is G.layout_tick and ev.graphmodel.build_knn_graph is G.build_knn_graph
        assert ev.graphmodel.kmeans_tick is G.kmeans_tick
    finally:
        sys.path.remove(str(src))
        for m in [m for m in sys.modules if m == "embedview" or m.startswith("embedview.")]:
            del sys.modules[m]
