"""Batch-SOM landmark training with point sharding across GPUs.

NEW relative to the reference, which trains online only (ref: som.py:44-68;
SPEC.md:270).  Semantics:

  1. b_i = exact f32 nearest landmark of x_i (the k-NN contract, k = 1)
  2. S_b = sum_{b_i = b} x_i (f64),  C_b = #{i : b_i = b}
  3. all-reduce (S, C) over the point shards (one NCCL call per step)
  4. H_jb = exp(-|lo_j - lo_b|^2 / (2 sigma^2)),  num = H S,  den = H C
  5. mean-field: hi_j += (alpha / B)(num_j - den_j hi_j)   (B = sum C; at B = 1
     this is som_tick's update for that sample), or Kohonen: hi_j = num_j / den_j.

The statistics are exact int64 fixed point (``acc_fx_bits`` fractional
bits, chosen once from the dataset's magnitude and size): integer sums do
not depend on accumulation order, atomic scheduling or how the points are
split over ranks, so the landmarks after any number of steps are
bit-identical at every GPU count (SURVEY §7 hard part 6).  They come from
the embed's k-NN (BMU = idx[:, 0]) as a separate pass over X: a shared-
memory table in natural point order when it fits one SM (C3), else segment
sums over the BMU-sorted order the projection also uses (C4).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .core import ParameterError, points_of
from .projection import PreparedModel

_MODES = {"mean_field": 0, "kohonen": 1}


@dataclass(frozen=True)
class BatchSomConfig:
    sigma: float = 1.0
    alpha: float = 0.1
    mode: str = "mean_field"

    def __post_init__(self):
        if not self.sigma > 0:
            raise ParameterError(f"sigma must be > 0, got {self.sigma}")
        if not 0.0 <= self.alpha <= 1.0:
            raise ParameterError(f"alpha must be in [0, 1], got {self.alpha}")
        if self.mode not in _MODES:
            raise ParameterError(f"unknown batch SOM mode {self.mode!r}")


def _allreduce_(buf: torch.Tensor, group=None) -> None:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


def acc_fx_bits(maxabs: float, n_total: int) -> int:
    """Fractional bits of the int64 fixed-point statistics: the most (capped at
    40, i.e. 9e-13 resolution) that keep n_total x max|x| x 2^fx below 2^61.
    Every rank must pass the GLOBAL max|x| and point count."""
    bound = float(n_total) * float(maxabs)
    if not math.isfinite(bound):
        raise ParameterError("non-finite points")
    if bound <= 0.0:
        return 40
    fx = int(math.floor(61.0 - math.log2(bound)))
    if fx < 0:
        raise ParameterError(f"point magnitudes too large for the fixed-point statistics (n x max|x| = {bound:.3g})")
    return min(40, fx)


def dataset_fx_bits(X: torch.Tensor, group=None) -> int:
    """acc_fx_bits of the points of all ranks (one amax pass + two tiny all-reduces)."""
    import torch.distributed as dist

    st = torch.stack([X.abs().amax().double() if X.numel() else torch.zeros((), dtype=torch.float64, device=X.device),
                      torch.tensor(float(X.shape[0]), dtype=torch.float64, device=X.device)])
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        mx, nn = st[:1].clone(), st[1:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(nn, op=dist.ReduceOp.SUM, group=group)
        st = torch.cat([mx, nn])
    mx, nn = st.tolist()
    return acc_fx_bits(mx, int(nn))


def new_acc(g: int, d: int, dev) -> torch.Tensor:
    """Packed statistics [S (g×d) | C (g)], int64 (one all-reduce per step)."""
    return torch.zeros(g * d + g, dtype=torch.int64, device=dev)


def update_landmarks_(hi: torch.Tensor, lo: torch.Tensor, acc: torch.Tensor, fx: int, cfg: BatchSomConfig) -> None:
    """In-place landmark update from packed int64 statistics acc = [S (g×d) | C (g)]."""
    g, d = hi.shape
    dev = hi.device
    _lib.call("esom_batch_som_update", _dev.ptr(acc), _dev.ptr(acc) + g * d * 8, int(fx), _dev.ptr(lo), g, d,
              float(cfg.sigma), float(cfg.alpha), _MODES[cfg.mode], _dev.ptr(hi), _dev.stream_handle(dev))


def accumulate(X: torch.Tensor, hi: torch.Tensor, acc: torch.Tensor, fx: int, qe_sum=None, flag=None) -> None:
    """acc += BMU statistics of device points X (no projection)."""
    n, d = X.shape
    g = hi.shape[0]
    dev = X.device
    ws = _dev.workspace(dev, _lib.load().esom_workspace_bytes(g, d, 1, 0), slot="bmu")
    _lib.call("esom_bmu_accumulate", _dev.ptr(X), n, d, _dev.ptr(hi), g, _dev.ptr(ws), ws.numel(), 0,
              _dev.ptr(acc), _dev.ptr(acc) + g * d * 8, int(fx), _dev.ptr(qe_sum), _dev.ptr(flag),
              _dev.stream_handle(dev))


def batch_som_step(dataset, model, cfg: BatchSomConfig, group=None):
    """One batch-SOM step over all points of ``dataset`` (this rank's shard
    when ``group`` spans several ranks); returns the new hi."""
    pts = points_of(dataset)
    want_numpy = not _dev.is_device_tensor(pts)
    dev = _dev.cuda_device(pts)
    with torch.cuda.device(dev):
        X = _dev.to_f32(pts, dev)
        hi = _dev.to_f32(model.hi, dev).clone()
        lo = _dev.to_f32(model.lo, dev)
        g, d = hi.shape
        acc = new_acc(g, d, dev)
        fx = dataset_fx_bits(X, group)
        flag = _dev.new_flag(dev)
        accumulate(X, hi, acc, fx, flag=flag)
        _dev.raise_if_nonfinite(flag)
        _allreduce_(acc, group)
        update_landmarks_(hi, lo, acc, fx, cfg)
        return _dev.out_like(hi, want_numpy)


class FrameLoop:
    """Device-resident interactive loop for one rank's shard of points.

    frame():  fused embed of the shard with BMU statistics under the current
    landmarks -> one all-reduce of [S | C] -> landmark update -> re-prepare
    (packed tiles + pair table) for the next frame.  With ``train=False`` a
    frame is the projection alone.  All launches are asynchronous on the
    current stream; nothing synchronizes with the host.
    """

    def __init__(self, X: torch.Tensor, hi, lo, k: int, cfg: BatchSomConfig | None = None, group=None,
                 train: bool = True):
        self.X = X
        self.dev = X.device
        self.cfg = cfg or BatchSomConfig()
        self.group = group
        self.train = train
        with torch.cuda.device(self.dev):
            # a private copy: training frames update the landmarks in place
            self.model = PreparedModel(_dev.to_f32(hi, self.dev).clone(), lo, k, device=self.dev)
            g, d = self.model.hi.shape
            self.acc = new_acc(g, d, self.dev)
            self.fx = dataset_fx_bits(X, group) if train else 0
            self.qe = torch.zeros(1, dtype=torch.float64, device=self.dev)
            self.xy = torch.empty((X.shape[0], 2), dtype=torch.float32, device=self.dev)
            self.flag = _dev.new_flag(self.dev)
            self.far = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # projection visiting order: nearest-landmark order pays off when most points
        # take the far-point path (trained SOMs; see DeviceSession._update_order);
        # decided from the first eager frames' census, then fixed (graph replays)
        self.bmu_order = False
        self._census_frames = 2

    @property
    def launches_per_frame(self) -> int:
        """Our own kernels per frame: the embed's k-NN + projection (per chunk),
        plus, when training, the landmark update and the model re-preparation
        (pack tiles, pair table, tensor-core operands)."""
        g, d = self.model.hi.shape
        n = self.X.shape[0]
        embed = _lib.load().esom_embed_launches(n, g, d, self.model.k)
        return embed + (4 if self.train else 0)

    def capture(self) -> "FrameLoop":
        """Record one frame as a CUDA graph (after a warm frame: workspaces
        allocated, kernel attributes set); frame() then replays it -- one
        graph launch instead of ~5-15 kernel launches and host calls per
        frame.  The library's launch counter only advances at capture, so the
        kernels per replay are kept in ``graph_launches``."""
        from . import _lib as L

        self._eager_frame()
        torch.cuda.synchronize(self.dev)
        if self._census_frames > 0:  # (eager frames before the capture may have decided it already:
            self._census()           # a second census here would read the zeroed counter)
        self._census_frames = 0
        n0 = L.load().esom_launch_count()
        g = torch.cuda.CUDAGraph()
        # thread_local: the NCCL watchdog thread (multi-rank runs) may touch the
        # CUDA runtime while this thread captures
        with torch.cuda.device(self.dev), torch.cuda.graph(g, capture_error_mode="thread_local"):
            self._eager_frame()
        self.graph_launches = L.load().esom_launch_count() - n0
        self.graph = g
        return self

    def frame(self) -> torch.Tensor:
        g = getattr(self, "graph", None)
        if g is not None:
            g.replay()
            return self.xy
        xy = self._eager_frame()
        if self._census_frames > 0:
            self._census_frames -= 1
            self._census()
        return xy

    def _far_arg(self):
        return self.far if self._census_frames > 0 else None

    def _census(self) -> None:
        """Far-point census of the last frame (one 4-byte read) -> visiting order."""
        self.bmu_order = 2 * int(self.far.item()) > self.X.shape[0]
        self.far.zero_()

    def _eager_frame(self) -> torch.Tensor:
        m = self.model
        g, d = m.hi.shape
        if not self.train:
            m.embed_into(self.X, self.xy, flag=self.flag, bmu_order=self.bmu_order, far_count=self._far_arg())
            return self.xy
        self.acc.zero_()
        self.qe.zero_()
        m.embed_into(self.X, self.xy, acc_S=self.acc, acc_C=self.acc[g * d:], acc_fx=self.fx, qe_sum=self.qe,
                     flag=self.flag, bmu_order=self.bmu_order, far_count=self._far_arg())
        _allreduce_(self.acc, self.group)
        update_landmarks_(m.hi, m.lo, self.acc, self.fx, self.cfg)
        m.update()  # re-pack tiles + pair table for the new landmarks
        return self.xy
