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


def install(embedview_module=None) -> None:
    """Reroute the reference's hot path to the B200 kernels.

    engine.py/cli.py import ``embed`` by name and call the trainers through
    their module attribute, so patching these names reroutes every caller.
    """
    import importlib

    ev = embedview_module or importlib.import_module("embedview")
    # submodules by import path: the package attribute ``knn`` is the function
    _gm, _knn, _proj, _som = (importlib.import_module(f"{__name__}.{m}")
                              for m in ("graphmodel", "knn", "projection", "som"))

    mods = {name: importlib.import_module(f"{ev.__name__}.{name}") for name in
            ("knn", "projection", "som", "graphmodel", "engine", "cli", "bench")}
    for name in ("knn", "knn_base", "knn_bitonic"):
        setattr(mods["knn"], name, getattr(_knn, name))
    mods["knn"]._BACKENDS.update({"base": _knn.knn_base, "bitonic": _knn.knn_bitonic})
    for name in ("embed", "project_neighbors", "project_point", "scores"):
        setattr(mods["projection"], name, getattr(_proj, name))
    mods["projection"].knn = _knn.knn
    for m in (mods["engine"], mods["cli"], mods["bench"]):
        if hasattr(m, "embed"):
            m.embed = _proj.embed
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
    mods["engine"].color_channel = _engine.color_channel
