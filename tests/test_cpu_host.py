"""CPU-only checks: the C-ABI library loads and exports every symbol of
include/esom.h, host-side validation mirrors the reference (raises before
any device work), the multi-rank statistics path (gloo, world size 2), and
the reference arm of bench.py."""
import json
import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "esom.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int32_t|int|size_t|void|double|const char \*)\s*\*?\s*(esom_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2201_00701_b200 import _lib

    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.esom_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), f"{s} not exported"
    # every ctypes signature corresponds to a declared symbol
    assert set(_lib.SIGNATURES) | set(_lib.HELPERS) == set(syms)


def test_library_is_sm100a():
    from paper_2201_00701_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "FFMA2" in sass and "FADD2" in sass  # packed f32x2 distance arithmetic
    assert "UBLKCP" in sass                     # TMA bulk copies staging the landmark tiles
    assert "UTCHMMA" in sass and "LDTM" in sass  # tcgen05.mma (split-bf16 screen) + TMEM loads


def test_host_validation_matches_reference():
    import paper_2201_00701_b200 as esom

    with pytest.raises(esom.ParameterError, match="violates"):
        esom.knn_base(np.ones((2, 2)), np.ones((3, 2)), 4)
    with pytest.raises(esom.ParameterError, match="power-of-two"):
        esom.knn_bitonic(np.ones((4, 2)), np.ones((32, 2)), 12)
    with pytest.raises(esom.ParameterError, match="unknown knn backend"):
        esom.knn(np.ones((4, 2)), np.ones((8, 2)), 4, backend="carrier-pigeon")
    with pytest.raises(esom.InputError, match="dimension mismatch"):
        esom.knn(np.ones((4, 3)), np.ones((8, 2)), 4)
    with pytest.raises(esom.ParameterError):
        esom.scores([1.0, 2.0])
    with pytest.raises(esom.InputError):
        esom.scores([1.0, 0.5, 2.0])
    model = esom.LandmarkModel.create(np.ones((8, 4), np.float32), np.zeros((8, 2), np.float32))
    with pytest.raises(esom.ParameterError):
        esom.embed(np.ones((3, 4)), model, esom.EmbedParams(k=16))
    with pytest.raises(esom.InputError):
        esom.embed(np.ones((3, 5)), model, esom.EmbedParams(k=4))
    with pytest.raises(esom.ParameterError):
        esom.SomConfig(sigma=0.0)
    with pytest.raises(esom.ParameterError):
        esom.KmeansConfig(alpha_km=0.0)
    with pytest.raises(esom.InputError):
        esom.Dataset.from_points(np.array([[np.nan]]))


def test_rng_matches_reference_stream(golden):
    from paper_2201_00701_b200.core import Rng

    assert np.array_equal(Rng(7).integers(0, 1 << 20, size=256), golden["c3_som_sample"])


_FX = 36  # fractional bits of the fixed-point statistics in the world-2 test


def _gloo_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    from oracle import oracle
    from paper_2201_00701_b200.batch_som import _allreduce_

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.load(ROOT / "tests" / "golden" / "golden.npz")
    pts, hi, lo = g["small_points"], g["small_hi0"], g["small_lo"]
    shard = np.array_split(np.arange(pts.shape[0]), world)[rank]
    fx = _FX
    S, C = oracle.batch_som_accumulate_fx(pts[shard], hi, fx)
    acc = torch.from_numpy(np.concatenate([S.ravel(), C]))  # int64 [S | C], as FrameLoop packs it
    _allreduce_(acc)  # the same call the device FrameLoop issues (NCCL there)
    gd = hi.size
    new_hi = oracle.batch_som_update_fx(acc[:gd].numpy().reshape(hi.shape), acc[gd:].numpy(), fx, lo, hi, 0.9, 0.3)
    if rank == 0:
        np.save(result_path, new_hi)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_batch_som_gloo_world2(tmp_path, golden):
    import torch.multiprocessing as mp
    from oracle import oracle

    port = 29500 + (os.getpid() % 1000)
    out = tmp_path / "hi.npy"
    mp.spawn(_gloo_worker, args=(2, port, str(out)), nprocs=2, join=True)
    sharded = np.load(out)
    pts, hi, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
    S, C = oracle.batch_som_accumulate_fx(pts, hi, _FX)
    whole = oracle.batch_som_update_fx(S, C, _FX, lo, hi, 0.9, 0.3)
    # exact integer statistics: the sharded step is bit-identical to the single-rank one
    assert np.array_equal(sharded, whole)
    # and the fixed-point rounding (2^-_FX) stays far inside f32 against the f64 restatement
    full = oracle.batch_som_step(pts, hi, lo, 0.9, 0.3)
    np.testing.assert_allclose(sharded, full, rtol=1e-6, atol=1e-7)


def test_acc_fx_bits_bounds():
    from paper_2201_00701_b200.batch_som import acc_fx_bits
    from paper_2201_00701_b200.core import ParameterError

    assert acc_fx_bits(0.0, 10) == 40 and acc_fx_bits(15.0, 10_000_000) == 33
    for mx, n in ((15.0, 10_000_000), (262144.0, 10_000_000), (1e-3, 1000)):
        fx = acc_fx_bits(mx, n)
        assert n * mx * 2.0 ** fx < 2.0 ** 62  # the int64 sum cannot overflow
    with pytest.raises(ParameterError):
        acc_fx_bits(1e30, 10)


def _gloo_gather_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    from paper_2201_00701_b200.core import Rng
    from paper_2201_00701_b200.sharded import gather_sample_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.load(ROOT / "tests" / "golden" / "golden.npz")
    pts = g["small_points"].copy()
    pts[3, 1] = -0.0  # signed zeros must survive the sum
    bounds = np.linspace(0, pts.shape[0], world + 1).astype(int)
    idx = Rng(11).integers(0, pts.shape[0], size=256)  # the same draw on every rank
    rows = gather_sample_rows(torch.from_numpy(pts[bounds[rank]:bounds[rank + 1]]), int(bounds[rank]),
                              np.concatenate([idx, [3]]))
    if rank == 0:
        np.save(result_path, rows.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_online_tick_rows_gloo_world2(tmp_path, golden):
    """Online ticks over sharded points: one all-reduce assembles the sampled
    rows bit-exactly on every rank."""
    import torch.multiprocessing as mp
    from oracle import oracle
    from paper_2201_00701_b200.core import Rng

    port = 30500 + (os.getpid() % 1000)
    out = tmp_path / "rows.npy"
    mp.spawn(_gloo_gather_worker, args=(2, port, str(out)), nprocs=2, join=True)
    rows = np.load(out)
    pts = golden["small_points"].copy()
    pts[3, 1] = -0.0
    idx = Rng(11).integers(0, pts.shape[0], size=256)
    want = pts[np.concatenate([idx, [3]])]
    assert rows.tobytes() == want.tobytes()
    hi, lo = golden["small_hi0"], golden["small_lo"]
    a = oracle.som_tick(rows[:256], hi, lo, np.arange(256), 0.9, 0.3)
    b = oracle.som_tick(pts, hi, lo, idx, 0.9, 0.3)
    assert np.array_equal(a, b)


def test_bench_reference_arm_runs_on_cpu():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["e2e"]["h2d_bytes_per_step"] == 0


def test_projection_system_equals_reference(golden):
    """projection_system is host-side f64 introspection (ref: projection.py:151-186,
    SURVEY §8a P4): identical to the reference's on the same inputs."""
    import importlib

    src = ROOT / "baseline" / "_ref"
    if not (src / "embedview").exists():
        pytest.skip("reference not staged")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(src))
    try:
        refp = importlib.import_module("embedview.projection")
        refc = importlib.import_module("embedview.core")
        from oracle import oracle
        from paper_2201_00701_b200.projection import projection_system

        pts, hi, lo = golden["small_points"], golden["small_hi0"], golden["small_lo"]
        idx, sqd = oracle.knn(pts[:40], hi, 8)
        sc = oracle.scores(sqd)
        model = refc.LandmarkModel.create(hi, lo)
        for i in range(40):
            a1, c1 = projection_system(pts[i], model, idx[i], sc[i])
            a2, c2 = refp.projection_system(pts[i], model, idx[i], refp.ScoreVector(scores=sc[i]))
            assert np.array_equal(a1, a2) and np.array_equal(c1, c2)
    finally:
        sys.path.remove(str(src))
        for m in [m for m in sys.modules if m == "embedview" or m.startswith("embedview.")]:
            del sys.modules[m]


def test_bench_rank_slices_tile_the_survey_dataset(monkeypatch):
    """bench.py's per-rank inputs: contiguous row blocks of ONE §8d dataset
    (same centres everywhere) and the same landmarks on every rank, drawn
    from the whole dataset (weak: n per rank; strong: the n rows split)."""
    import bench
    from paper_2201_00701_b200 import datagen

    monkeypatch.setitem(bench.WORKLOADS, "tw", (4, 3000, 5, 4, 4, 8, False, "weak", "test weak"))
    monkeypatch.setitem(bench.WORKLOADS, "ts", (4, 7001, 5, 4, 4, 8, True, "strong", "test strong"))
    for name, world, n_total in (("tw", 3, 9000), ("ts", 4, 7001)):
        full = datagen.gaussians(4, n_total, 5, seed=1)[0]
        hi_full, lo_full = datagen.som_model(full, 4, 4, seed=2)
        parts = []
        for r in range(world):
            pts, hi, lo, k, train, nt = bench.make_inputs(name, r, world)
            assert nt == n_total and np.array_equal(hi, hi_full) and np.array_equal(lo, lo_full)
            parts.append(pts)
        assert np.array_equal(np.concatenate(parts), full)
