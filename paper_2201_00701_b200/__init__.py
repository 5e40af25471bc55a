"""paper_2201_00701_b200 -- B200-native EmbedSOM hot path (arXiv 2201.00701).

Drop-in for the reference's CPU API (`embedview` knn / projection / som /
graphmodel hot-path functions): same names, arguments, array layouts and
errors, computed by hand-written sm_100a kernels in libesom.so through the
C ABI of include/esom.h.  See DESIGN.md.
"""

from .core import (  # noqa: F401
    BITONIC_K_CHOICES,
    Dataset,
    EmbedParams,
    InputError,
    LandmarkModel,
    ParameterError,
    Rng,
)
from .knn import NeighborList, knn, knn_base, knn_bitonic, sq_euclidean  # noqa: F401
from .projection import (  # noqa: F401
    PreparedModel,
    ScoreVector,
    embed,
    project_neighbors,
    project_point,
    projection_system,
    scores,
)
from .som import SomConfig, bmu, quantization_error, som_tick  # noqa: F401
from .graphmodel import KmeansConfig, kmeans_tick  # noqa: F401
from .batch_som import BatchSomConfig, FrameLoop, batch_som_step  # noqa: F401
from .engine import DeviceSession, FrameEngine, color_channel  # noqa: F401
from .io import DeviceDataset, TransformSpec, apply_transform, compute_dim_stats, load_fcs, parse_fcs  # noqa: F401
from .protocol import encode_frame_points  # noqa: F401
from .som import fit_hi_for_new_landmark  # noqa: F401
from .graphmodel import EdgeSet, LayoutState, build_knn_graph, layout_tick, net_forces  # noqa: F401

__version__ = "0.1.0"


def install(embedview_module=None, fast: bool = False) -> None:
    """Reroute the reference's hot path to the B200 kernels.

    engine.py/cli.py import ``embed`` by name and call the trainers through
    their module attribute, so patching these names reroutes every caller.

    By default the patched ``embed`` runs ``mode="faithful"`` (k-NN ->
    scores -> the reference's projection arithmetic op for op), so it equals
    ``project_point`` / ``project_neighbors`` exactly, as the reference's own
    tests expect (tests:test_projection.py:202-246).  ``fast=True`` installs
    the tolerance-checked fast projection (<= 1e-4 x extent) instead.
    """
    import importlib

    ev = embedview_module or importlib.import_module("embedview")
    # submodules by import path: the package attribute ``knn`` is the function
    _gm, _knn, _proj, _som = (importlib.import_module(f"{__name__}.{m}")
                              for m in ("graphmodel", "knn", "projection", "som"))

    mods = {name: importlib.import_module(f"{ev.__name__}.{name}") for name in
            ("core", "knn", "projection", "som", "graphmodel", "engine", "cli", "bench")}
    _adopt_reference_types(mods)
    for name in ("knn", "knn_base", "knn_bitonic"):
        setattr(mods["knn"], name, getattr(_knn, name))
    mods["knn"]._BACKENDS.update({"base": _knn.knn_base, "bitonic": _knn.knn_bitonic})
    embed_fn = _proj.embed if fast else _faithful_embed
    for name in ("project_neighbors", "project_point", "scores"):
        setattr(mods["projection"], name, getattr(_proj, name))
    mods["projection"].embed = embed_fn
    mods["projection"].knn = _knn.knn
    for m in (mods["engine"], mods["cli"], mods["bench"]):
        if hasattr(m, "embed"):
            m.embed = embed_fn
    if hasattr(mods["bench"], "knn"):
        mods["bench"].knn = _knn.knn
    if hasattr(mods["bench"], "project_neighbors"):
        mods["bench"].project_neighbors = _proj.project_neighbors
    mods["som"].som_tick = _som.som_tick
    mods["som"].quantization_error = _som.quantization_error
    mods["som"].fit_hi_for_new_landmark = _som.fit_hi_for_new_landmark
    mods["graphmodel"].kmeans_tick = _gm.kmeans_tick
    # landmark-side graph ops (§8f row 2): engine.py reaches them through the module attribute
    for name in ("build_knn_graph", "graph_scale_for_unit_rest", "net_forces", "layout_tick"):
        setattr(mods["graphmodel"], name, getattr(_gm, name))
    # Engine.tick (§8f row 1): dataset resident in HBM, full re-projection per frame
    from . import engine as _engine
    from .engine import gpu_tick

    mods["engine"].Engine.tick = gpu_tick
    # the reference engine's frame semantics stay its own unless fast=True: the
    # 131072-point round-robin refresh and the installed embed's arithmetic
    # (tests:test_engine.py:162-195 compare tick positions with embed() exactly)
    mods["engine"].Engine.full_reprojection = bool(fast)
    mods["engine"].Engine.embed_mode = "fast" if fast else "faithful"
    mods["engine"].color_channel = _engine.color_channel
    # the package-level re-exports (``embedview.embed`` etc., ref: __init__.py:22-34)
    for name, fn in (("knn", _knn.knn), ("knn_base", _knn.knn_base), ("knn_bitonic", _knn.knn_bitonic),
                     ("embed", embed_fn), ("project_point", _proj.project_point), ("scores", _proj.scores),
                     ("som_tick", _som.som_tick), ("quantization_error", _som.quantization_error),
                     ("fit_hi_for_new_landmark", _som.fit_hi_for_new_landmark),
                     ("kmeans_tick", _gm.kmeans_tick), ("build_knn_graph", _gm.build_knn_graph),
                     ("layout_tick", _gm.layout_tick)):
        if hasattr(ev, name):
            setattr(ev, name, fn)


def _faithful_embed(points, model, params, backend: str = "bitonic", chunk_size=None):
    """The reference's ``embed`` signature (ref: projection.py:220-245) bound
    to the bit-faithful projection mode (what ``install()`` patches in)."""
    from .projection import embed as _embed

    return _embed(points, model, params, backend=backend, chunk_size=chunk_size, mode="faithful")


def _adopt_reference_types(mods) -> None:
    """Make the installed functions speak the reference's types.

    * Errors: each core error class (``InputError``, ``ParameterError``,
      ``ParseError``) is replaced, in every module of this package, by a
      subclass of BOTH this package's class and the reference's, so what the
      B200 path raises is caught by ``except embedview.core.ParameterError``
      / ``pytest.raises(...)`` in the reference's callers and tests (ref:
      core.py:18-27; engine.py:352) as well as by this package's own class.
    * Result types: ``knn`` returns the reference's ``NeighborList`` and
      ``scores`` its ``ScoreVector`` (same frozen dataclass fields), so the
      reference's own helpers (``projection_system``'s isinstance check)
      accept them.
    """
    import sys

    from . import core as _core, knn as _knn, projection as _proj

    ref_core = mods["core"]
    swap = {}
    for name in ("InputError", "ParameterError", "ParseError"):
        ours, theirs = getattr(_core, name, None), getattr(ref_core, name, None)
        if ours is None or theirs is None or issubclass(ours, theirs):
            continue
        swap[ours] = type(name, (ours, theirs), {"__module__": ours.__module__, "__doc__": ours.__doc__})
    if swap:
        for mname, m in list(sys.modules.items()):
            if m is None or not (mname == __name__ or mname.startswith(__name__ + ".")):
                continue
            for attr, val in list(vars(m).items()):
                if isinstance(val, type) and val in swap:
                    setattr(m, attr, swap[val])
    _knn.NeighborList = mods["knn"].NeighborList
    _proj.ScoreVector = mods["projection"].ScoreVector
