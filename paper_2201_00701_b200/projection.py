"""Scores, projection and ``embed`` on the B200 (mirror of ref: projection.py).

* ``scores`` / ``project_point`` / ``project_neighbors`` run the faithful
  kernels: the reference's mixed f32/f64 arithmetic
  with every operation separately rounded, so results equal the reference
  except where CUDA's f64 ``exp`` differs from glibc's by one ulp.
* ``embed`` (``mode="fast"``, the default) runs, per chunk of points, the
  exact k-NN (d <= 32: tensor-core screen, BMU counting sort, exact
  re-evaluation; d > 32: operand split, tcgen05 GEMM screen, BMU sort, exact
  re-evaluation) and one projection kernel: scores in registers and each
  pair's high-dimensional coordinate through the law of cosines on the exact
  squared distances (no neighbour-row gathers; far points recompute their
  distances in f64), checked to the stated tolerance (max |xy - xy_ref| <=
  1e-4 x embedding extent).  ``esom_embed_launches`` counts the launches.
  ``mode="faithful"`` chains knn -> scores -> faithful projection instead
  (what ``install()`` patches into the reference by default).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .core import EmbedParams, InputError, ParameterError
from .knn import NeighborList, _run_knn, knn

SCORE_EPS = 1e-9   # ref: projection.py:25
PAIR_EPS = 1e-12   # ref: projection.py:26
DET_REL = 1e-9     # ref: projection.py:27
DET_ABS = 1e-30    # ref: projection.py:28


@dataclass(frozen=True)
class ScoreVector:
    """Non-negative weights aligned with one NeighborList row (ref: projection.py:31-35)."""

    scores: np.ndarray


def _scores_dev(sqd: torch.Tensor) -> torch.Tensor:
    dev = sqd.device
    n, k = sqd.shape
    out = torch.empty((n, k), dtype=torch.float64, device=dev)
    _lib.call("esom_scores", _dev.ptr(sqd), n, k, _dev.ptr(out), _dev.stream_handle(dev))
    return out


def scores(sqdists) -> ScoreVector:
    """One ascending row of squared distances -> scores (ref: projection.py:124-142)."""
    row = np.asarray(sqdists, dtype=np.float32).ravel()
    k = row.shape[0]
    if k < 3:
        raise ParameterError(f"need k >= 3 distances, got {k}")
    if np.any(row < 0) or not np.all(np.isfinite(row)):
        raise InputError("squared distances must be finite and non-negative")
    if np.any(np.diff(row) < 0):
        raise InputError("squared distances must be ascending")
    dev = _dev.cuda_device()
    with torch.cuda.device(dev):
        out = _scores_dev(_dev.to_f32(row.reshape(1, -1), dev))
        return ScoreVector(scores=out[0].cpu().numpy())


def projection_system(x_i, model, nbr_indices, s):
    """Normal equations (A, c) for one point, pure f64 (ref: projection.py:151-186).

    Host-side introspection helper (the reference's own f64 numpy routine);
    not part of the accelerated path.
    """
    hi = np.asarray(model.hi, np.float64)
    lo = np.asarray(model.lo, np.float64)
    x = np.asarray(x_i, np.float64).ravel()
    idx = np.asarray(nbr_indices, np.int64).ravel()
    sc = np.asarray(getattr(s, "scores", s), np.float64).ravel()
    a = np.zeros((2, 2))
    c = np.zeros(2)
    k = idx.shape[0]
    for u in range(k):
        if sc[u] <= 0:
            continue
        for v in range(u + 1, k):
            w = sc[u] * sc[v]
            if w <= 0:
                continue
            hd = hi[idx[v]] - hi[idx[u]]
            hd2 = hd @ hd
            if hd2 < PAIR_EPS:
                continue
            ld = lo[idx[v]] - lo[idx[u]]
            ld2 = ld @ ld
            if ld2 < PAIR_EPS:
                continue
            grad = ld / ld2
            h = ((x - hi[idx[u]]) @ hd) / hd2 + grad @ lo[idx[u]]
            a += w * np.outer(grad, grad)
            c += w * h * grad
    return a, c


def _model_arrays(model, dev):
    return _dev.to_f32(model.hi, dev), _dev.to_f32(model.lo, dev)


def _project_dev(X, hi, lo, idx, sc) -> torch.Tensor:
    dev = X.device
    n, d = X.shape
    k = idx.shape[1]
    xy = torch.empty((n, 2), dtype=torch.float32, device=dev)
    _lib.call("esom_project", _dev.ptr(X), n, d, _dev.ptr(hi), _dev.ptr(lo), hi.shape[0], _dev.ptr(idx),
              _dev.ptr(sc), k, _dev.ptr(xy), _dev.stream_handle(dev))
    return xy


def project_point(x_i, model, nbr_indices, s) -> np.ndarray:
    """Project one point from its neighbour row and scores (ref: projection.py:189-208)."""
    x = np.ascontiguousarray(np.asarray(x_i, dtype=np.float32)).reshape(1, -1)
    if x.shape[1] != model.hi.shape[1]:
        raise InputError(f"point has {x.shape[1]} dims, model expects {model.hi.shape[1]}")
    idx = np.ascontiguousarray(nbr_indices, dtype=np.int32).reshape(1, -1)
    sc = np.ascontiguousarray(np.asarray(getattr(s, "scores", s), np.float64)).reshape(1, -1)
    if idx.shape[1] != sc.shape[1]:
        raise InputError("neighbor row and score vector lengths differ")
    if idx.shape[1] < 3:
        raise ParameterError("projection needs k >= 3 neighbors")
    dev = _dev.cuda_device()
    with torch.cuda.device(dev):
        hi, lo = _model_arrays(model, dev)
        xy = _project_dev(_dev.to_f32(x, dev), hi, lo, _dev.to_i32(idx, dev), _dev.to_f64(sc, dev))
        return xy[0].cpu().numpy()


def project_neighbors(points, model, nbrs: NeighborList):
    """Scores + faithful projection over precomputed neighbour lists (ref: projection.py:211-217)."""
    want_numpy = not _dev.is_device_tensor(points)
    dev = _dev.cuda_device(points)
    with torch.cuda.device(dev):
        X = _dev.to_f32(points, dev)
        hi, lo = _model_arrays(model, dev)
        sqd = _dev.to_f32(nbrs.sqdists, dev)
        sc = _scores_dev(sqd)
        xy = _project_dev(X, hi, lo, _dev.to_i32(nbrs.indices, dev), sc)
        return _dev.out_like(xy, want_numpy)


class PreparedModel:
    """Device copy of (hi, lo) plus the fused kernel's workspace: packed
    landmark tiles (TMA source) and the g×g pair table.  Rebuild (``update``)
    whenever hi or lo changes; cheap (O(g^2 d))."""

    def __init__(self, hi, lo, k: int, device=None):
        self.device = device if device is not None else _dev.cuda_device(hi)
        self.k = int(k)
        self.update(hi, lo)

    def update(self, hi=None, lo=None):
        """Re-prepare after hi (and/or lo) changed.  The screen-row order
        derives from lo alone, so it is kept when no new lo is given."""
        dev = self.device
        with torch.cuda.device(dev):
            keep = lo is None and getattr(self, "ws", None) is not None
            if hi is not None:
                self.hi = _dev.to_f32(hi, dev)
            if lo is not None:
                self.lo = _dev.to_f32(lo, dev)
            self.g, self.d = self.hi.shape
            nbytes = _lib.load().esom_workspace_bytes(self.g, self.d, self.k, 1)
            if getattr(self, "ws", None) is None or self.ws.numel() < nbytes:
                self.ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
                keep = False
            if getattr(self, "flag", None) is None:
                self.flag = _dev.new_flag(dev)
            _lib.call("esom_prepare_model", _dev.ptr(self.hi), _dev.ptr(self.lo), self.g, self.d, self.k,
                      1 if keep else 0, _dev.ptr(self.ws),
                      self.ws.numel(), _dev.ptr(self.flag), _dev.stream_handle(dev))
        return self

    def point_workspace(self, n: int) -> torch.Tensor:
        nbytes = _lib.load().esom_point_workspace_bytes(n, self.d, self.k)
        pws = getattr(self, "pws", None)
        if pws is None or pws.numel() < nbytes:
            self.pws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self.pws

    def embed_into(self, X: torch.Tensor, xy: torch.Tensor, *, bmu=None, acc_S=None, acc_C=None, acc_fx: int = 0,
                   qe_sum=None, flag=None, stream=None, bmu_order: bool = False, far_count=None) -> None:
        """Asynchronous embed of device points X (n×d f32) into xy (n×2 f32):
        k-NN + projection kernels per L2-resident chunk.  ``acc_S`` / ``acc_C``
        (int64, nullable) receive the batch-SOM statistics in fixed point with
        ``acc_fx`` fractional bits.  ``bmu_order`` visits the projection in
        nearest-landmark order; ``far_count`` (device int32) accumulates the
        points that took the f64 far-point path."""
        n, d = X.shape
        st = stream if stream is not None else _dev.stream_handle(self.device)
        pws = self.point_workspace(n)
        _lib.call("esom_embed_prepared_ex", _dev.ptr(X), n, d, _dev.ptr(self.hi), _dev.ptr(self.lo), self.g, self.k,
                  _dev.ptr(self.ws), _dev.ptr(pws), pws.numel(), _dev.ptr(xy), _dev.ptr(bmu), _dev.ptr(acc_S),
                  _dev.ptr(acc_C), int(acc_fx), _dev.ptr(qe_sum), _dev.ptr(flag if flag is not None else self.flag),
                  1 if bmu_order else 0, _dev.ptr(far_count), st)


def embed(points, model, params: EmbedParams, backend: str = "bitonic", chunk_size: int | None = None,
          mode: str = "fast"):
    """Full pipeline -> n×2 f32 (ref: projection.py:220-245).

    Same validation and errors as the reference; output is chunk-invariant
    (``chunk_size`` only bounds device memory per launch).  Device tensors in
    -> device tensor out; numpy in -> numpy out.
    """
    ps = _dev.is_device_tensor(points) and tuple(points.shape) or np.shape(points)
    if len(ps) != 2:
        raise InputError("points must be a 2-d matrix")
    if ps[1] != model.hi.shape[1]:
        raise InputError(f"points have d={ps[1]}, model has d={model.hi.shape[1]}")
    g = model.hi.shape[0]
    params.validate(g, backend)
    if backend not in ("base", "bitonic"):
        raise ParameterError(f"unknown knn backend {backend!r}")
    k = params.k
    want_numpy = not _dev.is_device_tensor(points)
    dev = _dev.cuda_device(points)
    if mode == "fast" and k <= 64 and not chunk_size and ps[0] >= 2 * _pipe_chunk(g):
        host = _pipelinable_host(points)
        if host is not None:
            with torch.cuda.device(dev):
                return _embed_host_pipelined(host, model, k, dev)
    with torch.cuda.device(dev):
        X = _dev.to_f32(points, dev)
        n = X.shape[0]
        xy = torch.empty((n, 2), dtype=torch.float32, device=dev)
        if n == 0:
            return _dev.out_like(xy, want_numpy)
        step = n if not chunk_size else max(1, int(chunk_size))
        if mode == "faithful" or k > 64:
            hi, lo = _model_arrays(model, dev)
            for s in range(0, n, step):
                nb = _run_knn(X[s:s + step], hi, k)
                sc = _scores_dev(nb.sqdists)
                xy[s:s + step] = _project_dev(X[s:s + step], hi, lo, nb.indices, sc)
            return _dev.out_like(xy, want_numpy)
        if mode != "fast":
            raise ParameterError(f"unknown projection mode {mode!r}")
        try:
            pm = PreparedModel(model.hi, model.lo, k, device=dev)
            flag = _dev.new_flag(dev)
            for s in range(0, n, step):
                pm.embed_into(X[s:s + step], xy[s:s + step], flag=flag)
        except _lib.UnsupportedShape:
            # beyond the fast kernels' shared-memory plans (very large g): the
            # faithful chain covers any shape, like the reference
            return embed(X if not want_numpy else points, model, params, backend, chunk_size, mode="faithful")
        _dev.raise_if_nonfinite(flag)
        _dev.raise_if_nonfinite(pm.flag)
        return _dev.out_like(xy, want_numpy)


# points per H2D/compute/D2H stage (measured on B200, PCIe 54 GB/s each way: 2^17 best at
# g <= 256, 2^18 above, where each stage carries more fixed kernel work) and rotating buffers
PIPE_CHUNK = int(os.environ.get("ESOM_PIPE_CHUNK", 0)) or None
PIPE_DEPTH = int(os.environ.get("ESOM_PIPE_DEPTH", 3))


def _pipe_chunk(g: int) -> int:
    return PIPE_CHUNK or (1 << 17 if g <= 256 else 1 << 18)


def _pipelinable_host(points):
    """Host inputs the chunked pipeline takes: a pinned f32 torch tensor (DMA
    straight from it) or a C-contiguous f32 numpy array -- the reference's own
    calling convention -- staged through pinned chunks.  Anything else (other
    dtypes, strided arrays) takes the one-shot conversion path."""
    if isinstance(points, torch.Tensor):
        if (not points.is_cuda and points.dtype == torch.float32 and points.is_contiguous()
                and points.is_pinned()):
            return points
        return None
    if isinstance(points, np.ndarray) and points.dtype == np.float32 and points.flags.c_contiguous:
        pinned = _pinned_in_place(points)
        return pinned if pinned is not None else points
    return None


# numpy inputs embedded repeatedly (the interactive loop re-projects the same
# dataset every frame) are pinned IN PLACE on their second use
# (cudaHostRegister), so later calls DMA straight from the caller's array at
# full PCIe speed; the range is unpinned when the array is garbage collected.
# One-shot inputs keep the staged copy (registration costs about as much as
# the copy).  Bounded by _HOST_REG_CAP bytes.
_HOST_REG: dict = {}
_HOST_SEEN: dict = {}
_HOST_REG_CAP = 16 << 30
_HOST_LOCK = None


def _pinned_in_place(host: np.ndarray):
    import threading
    import weakref

    global _HOST_LOCK
    if _HOST_LOCK is None:
        _HOST_LOCK = threading.Lock()
    ptr = int(host.__array_interface__["data"][0])
    key = (ptr, int(host.nbytes))
    owner = host
    while isinstance(owner.base, np.ndarray):
        owner = owner.base
    if owner.base is not None or host.nbytes < (8 << 20):
        return None  # foreign buffer (mmap, bytes, ...) or too small to matter
    with _HOST_LOCK:
        if key in _HOST_REG:
            return torch.from_numpy(host)
        oid = id(owner)
        if _HOST_SEEN.get(key) != oid:  # first use: remember, copy through staging
            _HOST_SEEN.clear()
            _HOST_SEEN[key] = oid
            return None
        if sum(k[1] for k in _HOST_REG) + key[1] > _HOST_REG_CAP:
            return None
        if _lib.load().esom_host_register(ptr, key[1]) != 0:
            return None  # (already registered by someone else, or no memory to lock)

        def _release(k=key):
            with _HOST_LOCK:
                if _HOST_REG.pop(k, None) is not None:
                    _lib.load().esom_host_unregister(k[0])

        _HOST_REG[key] = weakref.finalize(owner, _release)
    return torch.from_numpy(host)


def _embed_host_pipelined(host, model, k: int, dev) -> np.ndarray:
    """embed() for host points: chunked H2D on one copy stream, the kernels on
    the compute stream and the D2H of finished chunks on a second copy stream
    (PCIe is full duplex), with PIPE_DEPTH rotating device buffers, so the end
    -to-end time approaches max(H2D, compute) instead of their sum.  A numpy
    input (pageable) is first copied by host threads into a ring of pinned
    staging chunks (a chunk is rewritten only after its previous H2D ran).
    (A ramp of smaller first stages measured slower: the fixed per-stage
    cost outweighs the shorter pipeline fill.)"""
    try:
        return _embed_host_pipeline_run(host, model, k, dev)
    except _lib.UnsupportedShape:
        # beyond the fast kernels' shared-memory plans: the faithful chain (any shape)
        torch.cuda.synchronize(dev)
        return embed(host if isinstance(host, np.ndarray) else host.numpy(), model, EmbedParams(k=k), mode="faithful")


def _embed_host_pipeline_run(host, model, k: int, dev) -> np.ndarray:
    n, d = host.shape
    flag = _dev.new_flag(dev)
    out = torch.empty((n, 2), dtype=torch.float32, pin_memory=True)
    comp = torch.cuda.current_stream(dev)
    h2d, d2h = _copy_streams(dev)
    c = min(_pipe_chunk(model.hi.shape[0]), n)
    nb = PIPE_DEPTH
    Xd, Yd, fresh = _pipe_buffers(dev, nb, c, d)
    staged = isinstance(host, np.ndarray)
    if staged:
        stage = _pinned_stage(nb, c, d)
        stage_free = [None] * nb  # H2D that last read stage slot b
    if fresh:
        h2d.wait_stream(comp)  # new allocations: order after prior work on the compute stream
    loaded = [torch.cuda.Event() for _ in range(nb)]
    computed = [None] * nb  # compute of the chunk that last used buffer b (Xd[b] free, Yd[b] ready)
    drained = [None] * nb   # D2H of the chunk that last used buffer b (Yd[b] free)
    starts = list(range(0, n, c))

    def load(it):  # H2D of chunk it into buffer it % nb (after that buffer's previous compute)
        s = starts[it]
        m = min(c, n - s)
        b = it % nb
        if computed[b] is not None:
            h2d.wait_event(computed[b])
        if staged:
            if stage_free[b] is not None:
                stage_free[b].synchronize()
            _host_copy(stage[b][:m].numpy(), host[s:s + m])
            src = stage[b][:m]
        else:
            src = host[s:s + m]
        with torch.cuda.stream(h2d):
            Xd[b][:m].copy_(src, non_blocking=True)
        loaded[b].record(h2d)
        if staged:
            stage_free[b] = loaded[b]

    load(0)  # the first chunk's H2D runs while the model is prepared (host + device)
    pm = PreparedModel(model.hi, model.lo, k, device=dev)
    for it, s in enumerate(starts):
        if it + 1 < len(starts):
            load(it + 1)
        m = min(c, n - s)
        b = it % nb
        comp.wait_event(loaded[b])
        if drained[b] is not None:
            comp.wait_event(drained[b])
        pm.embed_into(Xd[b][:m], Yd[b][:m], flag=flag)
        ev = torch.cuda.Event()
        ev.record(comp)
        computed[b] = ev
        d2h.wait_event(ev)
        with torch.cuda.stream(d2h):
            out[s:s + m].copy_(Yd[b][:m], non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(d2h)
        drained[b] = ev2
    d2h.synchronize()
    comp.synchronize()
    _dev.raise_if_nonfinite(flag)
    _dev.raise_if_nonfinite(pm.flag)
    return out.numpy()


_COPY_POOL = None


def _host_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """Pageable -> pinned copy of one stage, split over host threads (numpy
    releases the GIL inside the copy loop)."""
    global _COPY_POOL
    parts = 4
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(parts, thread_name_prefix="esom-stage")
    m = src.shape[0]
    step = (m + parts - 1) // parts
    futs = [_COPY_POOL.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, m, step)]
    for f in futs:
        f.result()


def _pinned_stage(nb: int, c: int, d: int):
    """Pinned host staging ring of the numpy-input pipeline, per thread."""
    cache = getattr(_dev._tls, "pinned_stage", None)
    key = (nb, c, d)
    if cache is None or cache[0] != key:
        cache = _dev._tls.pinned_stage = (key, [torch.empty((c, d), dtype=torch.float32, pin_memory=True)
                                                for _ in range(nb)])
    return cache[1]


def _pipe_buffers(dev, nb: int, c: int, d: int):
    """Device staging buffers of the host pipeline, kept across calls per
    (thread, device) -- two threads embedding pinned inputs on one device
    never share them; the synchronous return of the pipeline guarantees the
    calling thread's buffers are idle."""
    cache = getattr(_dev._tls, "pipe_bufs", None)
    if cache is None:
        cache = _dev._tls.pipe_bufs = {}
    key = (str(dev), nb, c, d)
    fresh = key not in cache
    if fresh:
        cache.clear()
        cache[key] = ([torch.empty((c, d), dtype=torch.float32, device=dev) for _ in range(nb)],
                      [torch.empty((c, 2), dtype=torch.float32, device=dev) for _ in range(nb)])
    Xd, Yd = cache[key]
    return Xd, Yd, fresh


def _copy_streams(dev):
    """H2D and D2H copy streams of the host pipeline, per (thread, device)."""
    cache = getattr(_dev._tls, "copy_streams", None)
    if cache is None:
        cache = _dev._tls.copy_streams = {}
    key = (dev.index if isinstance(dev, torch.device) else int(dev))
    if key not in cache:
        cache[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return cache[key]
