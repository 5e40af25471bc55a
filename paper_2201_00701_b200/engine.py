"""Device-resident frame loop: the per-frame work of ``Engine.tick`` on the
B200 (ref: engine.py:347-399).

The reference tick drains commands, advances the online trainer, re-embeds
(131072-point round-robin chunks above that size) and emits a FramePacket,
re-uploading nothing only because it never leaves the host.  Here the
dataset is uploaded ONCE per dataset object and stays in HBM; per frame:

  trainer tick (host-drawn Philox samples, one CTA)  -> new hi
  model preparation (packed tiles, pair table)       -> one small launch set
  full re-projection of all n points                 -> tensor-core k-NN + projection
  colours (once per colour dimension)                -> esom_color_channel
  FramePoints record                                  -> esom_frame_points_pack
                                                        straight into pinned host memory

``DeviceSession`` holds that state for one dataset; ``FrameEngine`` is the
reference Engine's construction + SOM-mode tick without the command plane;
``gpu_tick`` is a drop-in replacement for ``embedview.engine.Engine.tick``
(installed by ``paper_2201_00701_b200.install``) that keeps the reference's
command handling, graph bookkeeping and packet type and moves the rest here.
"""

from __future__ import annotations

import sys
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .core import BITONIC_K_CHOICES, EmbedParams, InputError, LandmarkModel, ParameterError, Rng, points_of
from .graphmodel import KmeansConfig, kmeans_tick
from .knn import _run_knn
from .projection import PreparedModel
from .protocol import FrameBuffer, frame_points_bytes, pack_frame_points
from .som import SomConfig, som_tick

DEFAULT_CHUNK_SIZE = 131072  # ref: engine.py:31
MODE_SOM = "som"  # ref: engine.py:33-34
MODE_GRAPH = "graph"


def _nearest_pow2_k(requested: int, g: int) -> int:
    """ref: engine.py:156-160"""
    valid = [c for c in BITONIC_K_CHOICES if c <= g]
    if not valid:
        raise ParameterError(f"model too small for the bitonic backend (g={g})")
    return min(valid, key=lambda c: (abs(c - requested), c))


def _lattice(rows: int, cols: int) -> np.ndarray:
    ys, xs = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    return np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.float32)


def init_model(points, rng: Rng, grid=(16, 16), random_g=None) -> LandmarkModel:
    """The reference Engine's model initialisation (ref: engine.py:211-233):
    lattice (or uniform random) layout, hi = distinct dataset rows drawn
    from the session Rng."""
    n = points.shape[0]
    if grid is not None:
        rows, cols = grid
        if rows < 1 or cols < 1:
            raise ParameterError(f"bad grid {rows}x{cols}")
        g = rows * cols
        lo = _lattice(rows, cols)
    elif random_g is not None:
        g = int(random_g)
        if g < 4:
            raise ParameterError("need at least 4 landmarks")
        lo = rng.uniform(0.0, 1.0, size=(g, 2)).astype(np.float32)
    else:
        raise ParameterError("InitModel needs a grid or a landmark count")
    hi_idx = rng.choice_distinct(n, g)
    if isinstance(points, torch.Tensor):
        hi = points[torch.as_tensor(hi_idx, device=points.device)].float().cpu().numpy()
    else:
        hi = np.asarray(points)[hi_idx].astype(np.float32)
    return LandmarkModel.create(hi, lo)


def color_channel(dataset, color_dim: int):
    """Min-max quantise one dimension to u8, constant columns -> 128
    (ref: engine.py:144-153), on the device.  numpy in -> numpy out."""
    pts = points_of(dataset)
    sess = DeviceSession(dataset)
    out = sess.colors(color_dim)
    return out if _dev.is_device_tensor(pts) else out.cpu().numpy()


class _TrainModel:
    """hi (host or device) + lo, the two fields the trainers read."""

    def __init__(self, hi, lo):
        self.hi, self.lo = hi, lo


class _DeviceDataset:
    """Duck-typed dataset whose points are the session's device matrix."""

    def __init__(self, X: torch.Tensor):
        self.points = X


class DeviceSession:
    """HBM-resident state of one dataset's frames: the points (uploaded once),
    the prepared model, positions, colours and the pinned frame buffer."""

    def __init__(self, dataset, device=None):
        pts = points_of(dataset)
        self.source = dataset
        self.device = device if device is not None else _dev.cuda_device(pts)
        with torch.cuda.device(self.device):
            X = _dev.to_f32(pts, self.device)
            if X.ndim != 2 or X.shape[0] < 1 or X.shape[1] < 1:
                raise InputError("empty dataset")
            self.X = X
            self.n, self.d = X.shape
            self.positions = torch.zeros((self.n, 2), dtype=torch.float32, device=self.device)
            self.flag = _dev.new_flag(self.device)
            self.far_count = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._far_rows = 0  # rows embedded since far_count was last read
        self._far_host, self._far_ev, self._far_n = None, None, 0
        self.bmu_order = False
        self.data = _DeviceDataset(self.X)
        stats = getattr(dataset, "dim_stats", None)
        if stats is not None:  # the reference Dataset carries exact numpy statistics
            self.col_min = np.asarray(stats.min, dtype=np.float64)
            self.col_max = np.asarray(stats.max, dtype=np.float64)
        else:
            from .io import compute_dim_stats

            s = compute_dim_stats(self.X)
            self.col_min, self.col_max = s.min, s.max
        self._colors: dict[int, torch.Tensor] = {}
        self._pm: PreparedModel | None = None
        self._pm_key = None
        self._frame: FrameBuffer | None = None
        self._pos_host: torch.Tensor | None = None

    # -- per-frame pieces ---------------------------------------------------

    def colors(self, color_dim: int) -> torch.Tensor:
        """Device u8 colours of one dimension (ref: engine.py:144-153), cached."""
        if not 0 <= color_dim < self.d:
            raise ParameterError(f"color_dim={color_dim} out of range for d={self.d}")
        c = self._colors.get(color_dim)
        if c is None:
            with torch.cuda.device(self.device):
                c = torch.empty(self.n, dtype=torch.uint8, device=self.device)
                lo = float(self.col_min[color_dim])
                span = float(self.col_max[color_dim]) - lo  # f64, as the reference forms it
                _lib.call("esom_color_channel", _dev.ptr(self.X), self.n, self.d, int(color_dim), lo, span,
                          _dev.ptr(c), _dev.stream_handle(self.device))
            self._colors[color_dim] = c
        return c

    def train(self, trainer: str, model, cfg, rng) -> torch.Tensor:
        """One online trainer tick on the resident points; returns device hi."""
        with torch.cuda.device(self.device):
            if trainer == MODE_SOM:
                return som_tick(self.data, model, cfg, rng)
            return kmeans_tick(self.data, model, cfg, rng)

    def prepared(self, hi, lo, k: int) -> PreparedModel:
        if self._pm is None or self._pm.k != k or self._pm.hi.shape != tuple(np.shape(hi)):
            self._pm = PreparedModel(hi, lo, k, device=self.device)
        elif self._pm_key is None or self._pm_key[0] is not hi or self._pm_key[1] is not lo:
            self._pm.update(hi, lo)
        self._pm_key = (hi, lo)  # the objects themselves: identity, never a recycled id()
        return self._pm

    def embed(self, hi, lo, params: EmbedParams, backend: str = "bitonic", start: int = 0, stop=None,
              mode: str = "fast") -> torch.Tensor:
        """Re-project rows [start, stop) of the resident points (all by default).
        ``mode="faithful"``: k-NN -> scores -> the reference's projection
        arithmetic op for op (what ``embed(mode="faithful")`` computes)."""
        g = int(np.shape(hi)[0])
        params.validate(g, backend)
        if backend not in ("base", "bitonic"):
            raise ParameterError(f"unknown knn backend {backend!r}")
        stop = self.n if stop is None else stop
        if mode == "faithful":
            from .projection import _project_dev, _scores_dev

            with torch.cuda.device(self.device):
                if stop > start:
                    H, Lo = _dev.to_f32(hi, self.device), _dev.to_f32(lo, self.device)
                    Xs = self.X[start:stop]
                    nb = _run_knn(Xs, H, params.k)
                    self.positions[start:stop] = _project_dev(Xs, H, Lo, nb.indices, _scores_dev(nb.sqdists))
            return self.positions
        if mode != "fast":
            raise ParameterError(f"unknown projection mode {mode!r}")
        with torch.cuda.device(self.device):
            self._update_order()
            pm = self.prepared(hi, lo, params.k)
            if stop > start:
                pm.embed_into(self.X[start:stop], self.positions[start:stop], flag=self.flag,
                              bmu_order=self.bmu_order, far_count=self.far_count)
                self._far_rows += stop - start
        return self.positions

    def _update_order(self) -> None:
        """Visit the projection in nearest-landmark order when most points of
        the previous frame took the f64 far-point path (a trained SOM packs
        its landmarks tightly: neighbour rows are then shared across a warp,
        0.80 -> 0.61 ms per 2^20 points on C3; an untrained model skips the
        sort).  The census travels by an asynchronous 4-byte copy and is
        read once it has landed: the host never waits for it."""
        if self._far_rows and self._far_ev is None:
            st = torch.cuda.current_stream(self.device)
            if self._far_host is None:
                self._far_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            self._far_host.copy_(self.far_count, non_blocking=True)
            self.far_count.zero_()
            self._far_ev = torch.cuda.Event()
            self._far_ev.record(st)
            self._far_n, self._far_rows = self._far_rows, 0
        if self._far_ev is not None and self._far_ev.query():
            self.bmu_order = 2 * int(self._far_host.item()) > self._far_n
            self._far_ev = None

    def positions_host(self) -> np.ndarray:
        """Positions copied to a fresh host array (synchronises; raises on
        non-finite landmarks, like the reference's validation)."""
        with torch.cuda.device(self.device):
            if self._pos_host is None:
                self._pos_host = torch.empty((self.n, 2), dtype=torch.float32, pin_memory=True)
            self._pos_host.copy_(self.positions, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            self._check_flag()
            return self._pos_host.numpy().copy()

    def _check_flag(self) -> None:
        if int(self.flag.item()):
            self.flag.zero_()  # report once; the next frame starts clean
            raise InputError("non-finite input")

    def frame_record(self, frame_id: int, color_dim: int) -> memoryview:
        """The FramePoints wire record of the current positions, packed by the
        device into pinned host memory (ref: protocol.py:205-210).  The view
        is valid until the next call."""
        col = self.colors(color_dim)
        with torch.cuda.device(self.device):
            if self._frame is None:
                self._frame = FrameBuffer(frame_points_bytes(self.n), self.device)
            nbytes = pack_frame_points(self.positions, col, frame_id, self._frame)
            self._frame.event.synchronize()
            self._check_flag()
            return memoryview(self._frame.host.numpy())[:nbytes]


@dataclass(frozen=True)
class DeviceFrame:
    """What one FrameEngine tick emits (the reference FramePacket's fields;
    positions/colours stay on the device until asked for)."""

    frame_id: int
    positions: torch.Tensor
    landmarks_lo: np.ndarray
    landmark_ids: tuple
    colors: torch.Tensor


@dataclass
class FrameEngine:
    """The reference Engine's construction and SOM-mode tick with the
    dataset, model and frame resident on the B200 (ref: engine.py:163-199,
    347-399).  Graph mode (k-means + layout) and the command plane run
    through the reference Engine with ``gpu_tick`` installed."""

    dataset: object
    seed: int
    k: int = 16
    mode: str = MODE_SOM
    grid: tuple | None = (16, 16)
    random_g: int | None = None
    backend: str = "bitonic"
    color_dim: int = 0
    som_cfg: SomConfig = field(default_factory=SomConfig)
    km_cfg: KmeansConfig = field(default_factory=KmeansConfig)
    training_paused: bool = False

    pipelined: bool = True

    def __post_init__(self):
        if self.mode not in (MODE_SOM, MODE_GRAPH):
            raise ParameterError(f"unknown mode {self.mode!r}")
        if self.mode == MODE_GRAPH:
            raise ParameterError("graph mode (k-means + force layout) runs through the reference Engine "
                                 "with gpu_tick installed")
        self.rng = Rng(self.seed)
        self.session = DeviceSession(self.dataset)
        self._model = init_model(self.session.X, self.rng, self.grid, self.random_g)
        self.embed_params = EmbedParams(k=_nearest_pow2_k(self.k, self._model.g))
        self.frame_id = 0
        self._hi_dev = None   # device hi after the last training tick
        self._stale = False   # _model.hi lags _hi_dev
        self._spec = None     # speculative next tick (key, hi, done event, rng state)
        self._side = torch.cuda.Stream(self.session.device) if self.pipelined else None

    # the reference-facing model (numpy hi materialised on demand: one sync)
    @property
    def model(self) -> LandmarkModel:
        if self._stale:
            self._model = self._model.with_hi(self._hi_dev.cpu().numpy())
            self._stale = False
        return self._model

    @model.setter
    def model(self, m: LandmarkModel) -> None:
        self._drop_spec()
        self._model, self._hi_dev, self._stale = m, None, False

    def _train_input(self):
        hi = self._hi_dev if self._hi_dev is not None else self._model.hi
        return _TrainModel(hi, self._model.lo)

    def _drop_spec(self) -> None:
        """Discard a speculative tick: wait for it, rewind the Rng to before its draw."""
        if self._spec is not None:
            _, _, done, state = self._spec
            done.synchronize()
            self.rng._gen.bit_generator.state = state
            self._spec = None

    def tick(self) -> DeviceFrame:
        s = self.session
        if not self.training_paused:
            hi_new = None
            spec = self._spec
            key = spec[0] if spec is not None else None
            if key is not None and key[0] is self._hi_dev and key[1] == self.som_cfg and key[2] is self._model.lo:
                self._spec = None
                torch.cuda.current_stream(s.device).wait_event(spec[2])
                hi_new = spec[1]
            else:
                self._drop_spec()
                hi_new = s.train(MODE_SOM, self._train_input(), self.som_cfg, self.rng)
            self._hi_dev, self._stale = hi_new, True
        hi = self._hi_dev if self._hi_dev is not None else self._model.hi
        s.embed(hi, self._model.lo, self.embed_params, self.backend)
        if self._side is not None and not self.training_paused and self._spec is None:
            # the next tick's training depends only on this tick's hi: run it on a
            # side stream (one SM cluster) while the embed fills the GPU; same draws,
            # same order, rewound if anything changes before it is consumed
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(s.device))
            state = self.rng._gen.bit_generator.state
            with torch.cuda.stream(self._side):
                self._side.wait_event(ready)
                nxt = s.train(MODE_SOM, self._train_input(), self.som_cfg, self.rng)
                done = torch.cuda.Event()
                done.record(self._side)
            nxt.record_stream(torch.cuda.current_stream(s.device))
            self._spec = ((self._hi_dev, self.som_cfg, self._model.lo), nxt, done, state)
        self.frame_id += 1
        return DeviceFrame(frame_id=self.frame_id, positions=s.positions, landmarks_lo=self._model.lo,
                           landmark_ids=self._model.ids, colors=s.colors(self.color_dim))

    def frame_record(self) -> memoryview:
        """Wire bytes of the last frame (protocol.encode(FramePoints(...)))."""
        return self.session.frame_record(self.frame_id, self.color_dim)


# ---------------------------------------------------------------------------
# Drop-in Engine.tick for the reference engine (installed by install()).


def _session(engine) -> DeviceSession:
    ds = engine.state.dataset
    sess = getattr(engine, "_b200_session", None)
    if sess is None or sess.source is not ds:
        sess = DeviceSession(ds)
        engine._b200_session = sess
    return sess


def _spec_key(st, som: bool, sess) -> tuple:
    """What a speculative tick depended on: the hi array (and lo for SOM), the
    config, the mode and the dataset (compared by identity / equality)."""
    return (st.model.hi, st.model.lo if som else None, st.som_cfg if som else st.km_cfg, som, sess)


def _same_key(a, b) -> bool:
    return (a[0] is b[0] and a[1] is b[1] and a[2] == b[2] and a[3] == b[3] and a[4] is b[4])


def _rewind_spec(engine, spec) -> None:
    spec[2].synchronize()
    engine.state.rng._gen.bit_generator.state = spec[3]
    engine._b200_spec = None
    return None


def gpu_tick(self):
    """``Engine.tick`` with the dataset resident in HBM and a FULL
    re-projection every frame (ref: engine.py:347-399).  Command handling,
    graph-mode layout and the FramePacket type are the reference engine's
    own; set ``engine.full_reprojection = False`` to keep its 131072-point
    round-robin instead."""
    mod = sys.modules[type(self).__module__]
    st = self.state
    spec = getattr(self, "_b200_spec", None)
    if spec is not None and self._queue:
        spec = _rewind_spec(self, spec)  # commands may draw from st.rng: restore the draw order first
    for cmd in self._queue:
        try:
            self.apply_command(cmd)
        except (ParameterError, InputError, OSError, ValueError) as exc:
            self._errors.append(f"{type(exc).__name__}: {exc}")
    self._queue.clear()

    sess = _session(self)
    som = st.mode == mod.MODE_SOM
    if not st.training_paused:
        if spec is not None and _same_key(spec[0], _spec_key(st, som, sess)):
            self._b200_spec = None
            torch.cuda.current_stream(sess.device).wait_event(spec[2])
            hi = spec[1]
        else:
            if spec is not None:
                _rewind_spec(self, spec)
            hi = sess.train(MODE_SOM if som else "kmeans", st.model, st.som_cfg if som else st.km_cfg, st.rng)
        st.model = st.model.with_hi(hi.cpu().numpy())
        if getattr(self, "pipelined", True):
            # the next tick's training needs only this hi: run it on a side stream
            # during this frame's embed (rewound if a command or change intervenes)
            side = getattr(self, "_b200_side", None)
            if side is None:
                side = self._b200_side = torch.cuda.Stream(sess.device)
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(sess.device))
            state = st.rng._gen.bit_generator.state
            with torch.cuda.stream(side):
                side.wait_event(ready)
                nxt = sess.train(MODE_SOM if som else "kmeans", _TrainModel(hi, st.model.lo),
                                 st.som_cfg if som else st.km_cfg, st.rng)
                done = torch.cuda.Event()
                done.record(side)
            nxt.record_stream(torch.cuda.current_stream(sess.device))
            self._b200_spec = (_spec_key(st, som, sess), nxt, done, state)

    if st.mode == mod.MODE_GRAPH:
        if self._edges_dirty or self._ticks_since_rebuild >= mod.graphmodel.REBUILD_CADENCE:
            self._rebuild_edges()
        self._ticks_since_rebuild += 1
        pinned_rows = [st.model.ids.index(i) for i in st.model.pinned if i in st.model.ids]
        new_lo, vel = mod.graphmodel.layout_tick(st.model.lo, st.edges, st.layout, pinned_rows)
        st.model = st.model.with_lo(new_lo)
        st.layout = mod.replace(st.layout, velocities=vel)

    n = st.dataset.n
    if getattr(self, "full_reprojection", True) or n <= self.chunk_size:
        sess.embed(st.model.hi, st.model.lo, st.embed_params, self.backend, mode=getattr(self, "embed_mode", "fast"))
        st.chunk_cursor = 0
    else:
        if getattr(self, "_b200_positions", None) is not self._positions:
            sess.positions.zero_()  # the reference re-initialised its position buffer (ref: engine.py:229-230)
        start = st.chunk_cursor
        stop = min(start + self.chunk_size, n)
        sess.embed(st.model.hi, st.model.lo, st.embed_params, self.backend, start, stop,
                   mode=getattr(self, "embed_mode", "fast"))
        st.chunk_cursor = 0 if stop >= n else stop
    self._positions = self._b200_positions = sess.positions_host()

    st.frame_id += 1
    if self._colors is None:
        self._colors = sess.colors(st.color_dim).cpu().numpy()
    return mod.FramePacket(
        frame_id=st.frame_id,
        positions=self._positions,
        landmarks_lo=st.model.lo,
        landmark_ids=st.model.ids,
        edges=st.edges if st.mode == mod.MODE_GRAPH else mod.EdgeSet.empty(),
        colors=self._colors,
    )
