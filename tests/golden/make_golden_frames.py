"""Golden fixtures for the rows either side of the embed path:
frame colours, FramePoints wire records, FCS ingestion + transforms, the
reference Engine's SOM frames, and the landmark-side graph ops.  Made by
running the REFERENCE in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_frames.py

FCS files are written with the reference's own test writer
(tests/fcswriter.py of the reference) and stored as raw bytes, so nothing at
test time reads /root/reference.  Output: ``golden_frames.npz`` plus
``golden_frames.json`` (names, error cases, digests).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from embedview import graphmodel, protocol, som  # noqa: E402
from embedview.core import Dataset, LandmarkModel, ParseError  # noqa: E402
from embedview.datagen import extruded_s, gaussians  # noqa: E402
from embedview.engine import Engine, color_channel  # noqa: E402
from embedview.io import TransformSpec, apply_transform, parse_fcs  # noqa: E402
from fcswriter import write_fcs  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def main() -> None:
    arr: dict[str, np.ndarray] = {}
    meta: dict = {}
    rng = np.random.default_rng(20240817)  # tests:conftest.py:12-14 of the reference

    # -- colours (ref: engine.py:144-153) --------------------------------
    pts_s = extruded_s(800, seed=3)
    ds = Dataset.from_points(pts_s)
    arr["col_points"] = ds.points
    arr["col_colors"] = np.stack([color_channel(ds, c) for c in range(ds.d)])
    g_pts, _ = gaussians(8, 5000, 6, seed=1)
    g_pts = g_pts.astype(np.float32)
    g_pts[:, 3] = 2.5  # a constant column -> 128
    dg = Dataset.from_points(g_pts)
    arr["col2_points"] = dg.points
    arr["col2_colors"] = np.stack([color_channel(dg, c) for c in range(dg.d)])

    # -- FramePoints wire records (ref: protocol.py:205-210, 216-218) ------
    recs = []
    for i, n in enumerate((0, 1, 2, 3, 5, 7, 1000, 4099)):
        pos = rng.normal(0, 10, size=(n, 2)).astype(np.float32)
        col = rng.integers(0, 256, size=n).astype(np.uint8)
        fid = int(rng.integers(0, 2**32))
        rec = protocol.encode(protocol.FramePoints(frame_id=fid, positions=pos, colors=col))
        arr[f"rec{i}_pos"] = pos
        arr[f"rec{i}_col"] = col
        arr[f"rec{i}_bytes"] = np.frombuffer(rec, np.uint8)
        recs.append({"n": n, "frame_id": fid, "len": len(rec)})
    meta["records"] = recs

    # -- FCS parse (ref: io.py:72-126) -- tests:test_io.py:17-92 cases -----
    fcs = []

    def add_fcs(name, raw, expect_points=None):
        arr[f"fcs_{name}_raw"] = np.frombuffer(raw, np.uint8)
        ent = {"name": name}
        try:
            d = parse_fcs(raw)
            arr[f"fcs_{name}_points"] = d.points
            arr[f"fcs_{name}_min"] = d.dim_stats.min
            arr[f"fcs_{name}_max"] = d.dim_stats.max
            arr[f"fcs_{name}_mean"] = d.dim_stats.mean
            arr[f"fcs_{name}_sd"] = d.dim_stats.sd
            ent["names"] = list(d.dim_names)
            if expect_points is not None:
                assert np.array_equal(d.points, expect_points)
        except (ParseError, ValueError) as exc:
            ent["error"] = type(exc).__name__
            ent["message"] = str(exc)
        fcs.append(ent)

    add_fcs("small", write_fcs(rng.random((2, 3)).astype(np.float32), names=["FSC", "SSC", "CD4"]))
    for n in (1, 2, 1000):
        for d in (1, 8, 39):
            for bo in ("1,2,3,4", "4,3,2,1"):
                pts = (rng.random((n, d)) * 1000).astype(np.float32)
                add_fcs(f"grid_{n}_{d}_{'le' if bo[0] == '1' else 'be'}", write_fcs(pts, byteord=bo), pts)
    add_fcs("fcs31_text_offsets",
            write_fcs(rng.random((10, 4)).astype(np.float32), version=b"FCS3.1", offsets_in_text=True))
    add_fcs("doubled_delim", write_fcs(rng.random((3, 1)).astype(np.float32), names=["CD3/CD19"], delim=b"/"))
    add_fcs("lowercase_kw", write_fcs(rng.random((2, 1)).astype(np.float32)).replace(b"$DATATYPE", b"$DataType"))
    add_fcs("pns_name", write_fcs(rng.random((2, 1)).astype(np.float32), names=[""],
                                  extra_keywords={"$P1S": "Stain-A"}))
    add_fcs("bad_version", write_fcs(rng.random((1, 1)).astype(np.float32), version=b"FCS2.0"))
    add_fcs("bad_datatype", write_fcs(rng.random((1, 1)).astype(np.float32), datatype="I"))
    add_fcs("bad_byteord", write_fcs(rng.random((1, 1)).astype(np.float32), byteord="2,1,4,3"))
    add_fcs("bad_bits", write_fcs(rng.random((1, 2)).astype(np.float32), bits="16"))
    add_fcs("bad_mode", write_fcs(rng.random((1, 1)).astype(np.float32), mode="U"))
    add_fcs("truncated", write_fcs(rng.random((100, 4)).astype(np.float32))[:-50])
    add_fcs("missing_tot", write_fcs(rng.random((2, 1)).astype(np.float32)).replace(b"$TOT", b"$TXT"))
    add_fcs("short", b"FCS3.0   ")
    nan_pts = rng.random((4, 2)).astype(np.float32)
    nan_pts[2, 1] = np.nan
    add_fcs("nonfinite", write_fcs(nan_pts))
    big, _ = gaussians(16, 4000, 32, seed=5)
    add_fcs("cyto_be", write_fcs(big.astype(np.float32) * 100.0, byteord="4,3,2,1"))
    meta["fcs"] = fcs

    # -- transforms (ref: io.py:205-229), tests:test_io.py:157-219 ---------
    xf = []

    def add_xf(name, pts, entries):
        d = Dataset.from_points(pts)
        out = apply_transform(d, TransformSpec(entries=tuple(entries)))
        arr[f"xf_{name}_in"] = d.points
        arr[f"xf_{name}_out"] = out.points
        arr[f"xf_{name}_stats_in"] = np.stack([d.dim_stats.min, d.dim_stats.max, d.dim_stats.mean, d.dim_stats.sd])
        arr[f"xf_{name}_stats_out"] = np.stack(
            [out.dim_stats.min, out.dim_stats.max, out.dim_stats.mean, out.dim_stats.sd])
        xf.append({"name": name, "entries": [e if isinstance(e, str) else list(e) for e in entries]})

    add_xf("two_point", np.array([[0.0], [2.0]]), ["zscore"])
    add_xf("const_minmax", np.full((4, 1), 3.0), ["minmax"])
    add_xf("const_zscore", np.full((3, 1), 7.0), ["zscore"])
    add_xf("mixed", rng.random((100, 4)) * 10, ["none", "minmax", "zscore", ("affine", 2.0, -1.0)])
    add_xf("normal_z", rng.normal(3.0, 2.5, size=(500, 2)), ["zscore", "zscore"])
    add_xf("cyto_z", (big[:2000].astype(np.float32) * 100.0), ["zscore"] * 32)
    meta["transforms"] = xf

    # -- reference Engine, SOM mode (ref: engine.py:163-399) ---------------
    eng = Engine(ds, seed=99, k=16, grid=(6, 6))
    arr["eng_hi0"] = eng.state.model.hi
    arr["eng_lo"] = eng.state.model.lo
    ticks = []
    for t in range(6):
        p = eng.tick()
        arr[f"eng_pos{t}"] = p.positions
        arr[f"eng_hi{t + 1}"] = eng.state.model.hi
        rec = protocol.encode(protocol.FramePoints(frame_id=p.frame_id, positions=p.positions, colors=p.colors))
        ticks.append({"frame_id": p.frame_id, "record_sha": sha(rec), "len": len(rec)})
    arr["eng_colors"] = p.colors
    meta["engine"] = {"seed": 99, "k": 16, "grid": [6, 6], "n": 800, "ticks": ticks,
                      "k_eff": eng.state.embed_params.k}

    # -- landmark-side ops (ref: graphmodel.py:105-192, som.py:82-101) -----
    hi_g, lo_g = arr["eng_hi0"], arr["eng_lo"]
    edges = graphmodel.build_knn_graph(hi_g, 3, scale=1.0)
    arr["graph_pairs"] = edges.pairs
    arr["graph_rest"] = edges.rest
    st = graphmodel.LayoutState.for_count(hi_g.shape[0])
    st = graphmodel.replace(st, velocities=rng.normal(0, 0.1, size=(hi_g.shape[0], 2)))
    arr["layout_vel0"] = st.velocities
    lo_j = (lo_g + rng.normal(0, 0.05, size=lo_g.shape)).astype(np.float32)
    arr["layout_lo0"] = lo_j
    new_lo, vel = graphmodel.layout_tick(lo_j, edges, st, pinned_rows=[2, 7])
    arr["layout_forces"] = graphmodel.net_forces(lo_j, edges, st)
    arr["layout_lo1"] = new_lo
    arr["layout_vel1"] = vel
    meta["layout"] = {"stiffness": st.stiffness, "repulsion": st.repulsion, "damping": st.damping, "dt": st.dt,
                      "eps": graphmodel.REPULSION_EPS, "pinned": [2, 7]}
    model = LandmarkModel.create(hi_g, lo_g)
    fits = []
    for pos in ((2.5, 2.5), (0.0, 0.0), (5.0, 1.0), (-3.0, 9.0), (1.0 + 1e-4, 1.0)):
        fits.append(som.fit_hi_for_new_landmark(pos, model))
    arr["fit_pos"] = np.array([(2.5, 2.5), (0.0, 0.0), (5.0, 1.0), (-3.0, 9.0), (1.0 + 1e-4, 1.0)])
    arr["fit_hi"] = np.stack(fits)
    big_hi, _ = gaussians(16, 4096, 32, seed=7)
    e2 = graphmodel.build_knn_graph(big_hi.astype(np.float32), 8, scale=1.0)
    meta["graph4096_hi_sha"] = sha(np.ascontiguousarray(big_hi, np.float32).tobytes())  # regenerated in tests
    arr["graph4096_pairs"] = e2.pairs
    arr["graph4096_rest"] = e2.rest

    np.savez_compressed(OUT / "golden_frames.npz", **arr)
    (OUT / "golden_frames.json").write_text(json.dumps(meta, indent=1))
    print(f"wrote {len(arr)} arrays, {sum(a.nbytes for a in arr.values()) / 1e6:.1f} MB raw")


if __name__ == "__main__":
    main()
