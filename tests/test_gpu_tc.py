"""Tensor-core screened k-NN (esom_tc2.cuh pipelined screen with 2/3/4
warpgroups, and the round-streaming esom_tc.cuh): bit-identical to the
CUDA-core scan and to the reference oracle, including ties, on every
eligible shape."""
import os

import numpy as np
import pytest
import torch

from helpers import c1_inputs, c2_inputs
from oracle import oracle
import paper_2201_00701_b200 as esom

pytestmark = pytest.mark.gpu


def run(p, l, k, tc, w=None):
    """w: warpgroups of the split tc2 screen ("f<W>": the fused screen + exact kernel, 0: esom_tc.cuh)."""
    saved = {v: os.environ.get(v) for v in ("ESOM_TC", "ESOM_TC2_W", "ESOM_TC2_FUSED")}
    os.environ["ESOM_TC"] = "1" if tc else "0"
    if w is not None:
        w = str(w)
        if w.startswith("f"):
            os.environ["ESOM_TC2_FUSED"] = "1"
            w = w[1:]
        os.environ["ESOM_TC2_W"] = w
    try:
        nb = esom.knn_base(p, l, k)
    finally:
        for v, old in saved.items():
            if old is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = old
    return nb


@pytest.mark.parametrize("w", [3, 2, 4, "f4", "f3", 0])
@pytest.mark.parametrize("case", ["c1", "c2", "uniform16", "normal32", "ties", "wide", "rounds300", "c4like",
                                  "g4096", "ties777"])
def test_tc_equals_scan_and_oracle(case, w):
    gen = np.random.default_rng(hash(case) % 2**32)
    if case == "c1":
        p, l, _ = c1_inputs()
        k = 8
    elif case == "c2":
        p, l, _ = c2_inputs()
        p = p[: 1 << 17]
        k = 16
    elif case == "uniform16":
        p = gen.random((20000, 16)).astype(np.float32)
        l = gen.random((200, 16)).astype(np.float32)
        k = 16
    elif case == "normal32":
        p = (gen.normal(size=(20000, 32)) * 30 + 100).astype(np.float32)  # far from the origin
        l = (gen.normal(size=(256, 32)) * 30 + 100).astype(np.float32)
        k = 16
    elif case == "ties":
        p = gen.integers(0, 3, size=(20000, 8)).astype(np.float32)
        l = gen.integers(0, 3, size=(128, 8)).astype(np.float32)
        k = 16
    elif case == "wide":
        p = gen.normal(size=(5000, 5)).astype(np.float32) * np.float32(1e3)
        l = gen.normal(size=(37, 5)).astype(np.float32)
        k = 4
    elif case == "rounds300":  # two landmark rounds, the second partial
        p = gen.normal(size=(20000, 24)).astype(np.float32)
        l = gen.normal(size=(300, 24)).astype(np.float32)
        k = 16
    elif case == "c4like":
        from paper_2201_00701_b200 import datagen
        p = datagen.gaussians(16, 40000, 32, seed=3)[0]
        l = p[gen.choice(40000, 1024, replace=False)]
        k = 16
    elif case == "g4096":
        p = gen.random((8192, 16)).astype(np.float32)
        l = gen.random((4096, 16)).astype(np.float32)
        k = 8
    else:  # ties777
        p = gen.integers(0, 4, size=(10000, 6)).astype(np.float32)
        l = gen.integers(0, 4, size=(777, 6)).astype(np.float32)
        k = 16
    a = run(p, l, k, tc=True, w=w)
    b = run(p, l, k, tc=False)
    assert np.array_equal(a.indices, b.indices) and np.array_equal(a.sqdists, b.sqdists), case
    rows = np.arange(0, p.shape[0], max(1, p.shape[0] // 4000))
    wi, wd = oracle.knn(p[rows], l, k)
    assert np.array_equal(a.indices[rows], wi) and np.array_equal(a.sqdists[rows], wd), case


def test_tc_embed_and_stats_match_scan():
    p, hi, lo = c2_inputs()
    X = torch.from_numpy(p[: 1 << 18]).cuda()
    model = esom.LandmarkModel.create(hi, lo)
    os.environ["ESOM_TC"] = "1"
    xa = esom.embed(X, model, esom.EmbedParams(k=16))
    qa = esom.quantization_error(X, hi)
    os.environ["ESOM_TC"] = "0"
    xb = esom.embed(X, model, esom.EmbedParams(k=16))
    qb = esom.quantization_error(X, hi)
    del os.environ["ESOM_TC"]
    assert torch.equal(xa, xb)
    assert qa == pytest.approx(qb, rel=1e-12)


def run3(p, l, k, tc3):
    saved = os.environ.get("ESOM_TC3")
    os.environ["ESOM_TC3"] = "1" if tc3 else "0"
    try:
        return esom.knn_base(p, l, k)
    finally:
        if saved is None:
            os.environ.pop("ESOM_TC3", None)
        else:
            os.environ["ESOM_TC3"] = saved


@pytest.mark.parametrize("case", ["c5like", "d64_g257", "d100_ties", "d48_k5", "d512_uniform"])
def test_gemm_screen_equals_scan_and_oracle(case):
    """d > 32: tcgen05 GEMM screen (esom_tc3.cuh) + warp-exact re-evaluation."""
    gen = np.random.default_rng(abs(hash(case)) % 2**32)
    if case == "c5like":
        from paper_2201_00701_b200 import datagen
        p = datagen.gaussians(32, 1 << 15, 512, seed=5)[0]
        l = p[gen.choice(p.shape[0], 4096, replace=False)]
        k = 32
    elif case == "d64_g257":
        p = gen.random((20000, 64)).astype(np.float32)
        l = gen.random((257, 64)).astype(np.float32)
        k = 16
    elif case == "d100_ties":
        p = gen.integers(0, 3, size=(8000, 100)).astype(np.float32)
        l = gen.integers(0, 3, size=(300, 100)).astype(np.float32)
        k = 8
    elif case == "d48_k5":
        p = (gen.normal(size=(9000, 48)) * 20 + 50).astype(np.float32)
        l = (gen.normal(size=(700, 48)) * 20 + 50).astype(np.float32)
        k = 5
    else:
        p = gen.random((6000, 512)).astype(np.float32)
        l = gen.random((1000, 512)).astype(np.float32)
        k = 32
    a = run3(p, l, k, tc3=True)
    b = run3(p, l, k, tc3=False)
    assert np.array_equal(a.indices, b.indices) and np.array_equal(a.sqdists, b.sqdists), case
    rows = np.arange(0, p.shape[0], max(1, p.shape[0] // 500))
    wi, wd = oracle.knn(p[rows], l, k)
    assert np.array_equal(a.indices[rows], wi) and np.array_equal(a.sqdists[rows], wd), case


def test_gemm_exact_phase_unaligned_landmarks():
    """The grouped exact phase reads each lane's landmark-row sector with one
    256-bit load when the landmark matrix is 32-byte aligned, else with two
    128-bit loads: a landmark matrix at a 16-byte offset gives the same rows."""
    import torch
    gen = np.random.default_rng(11)
    p = (gen.normal(size=(5000, 64)) * 3).astype(np.float32)
    l = (gen.normal(size=(600, 64)) * 3).astype(np.float32)
    X = torch.from_numpy(p).cuda()
    buf = torch.zeros(l.size + 4, dtype=torch.float32, device="cuda")
    buf[4:] = torch.from_numpy(l.ravel()).cuda()
    H_off = buf[4:].view(l.shape)
    assert H_off.data_ptr() % 32 == 16
    H = torch.from_numpy(l).cuda()
    a = esom.knn(X, H, 32)
    b = esom.knn(X, H_off, 32)
    assert torch.equal(a.indices, b.indices) and torch.equal(a.sqdists, b.sqdists)
    rows = np.arange(0, p.shape[0], 37)
    wi, wd = oracle.knn(p[rows], l, 32)
    assert np.array_equal(b.indices.cpu().numpy()[rows], wi) and np.array_equal(b.sqdists.cpu().numpy()[rows], wd)
