"""pytest plugin: run the reference's OWN test suite with the B200 path installed.

Loaded with ``-p dropin_plugin`` by tests/test_gpu_dropin.py on the staged
copy of the reference's tests (baseline/_ref/embedview_tests, see
tools/stage_reference.sh).  At configure time -- before the reference's test
modules are imported, so their ``from embedview.knn import knn`` picks up the
patched names -- it calls ``esom.install(embedview)``, then records how many
of libesom's kernels ran during the session (``esom_launch_count``) and which
patched entry points were called, into the JSON file named by
``ESOM_DROPIN_REPORT``.
"""

from __future__ import annotations

import collections
import functools
import json
import os

_calls: collections.Counter = collections.Counter()
_state: dict = {}


def _counting(mod, name):
    fn = getattr(mod, name)

    @functools.wraps(fn)
    def wrapper(*a, **kw):
        _calls[f"{mod.__name__}.{name}"] += 1
        return fn(*a, **kw)

    setattr(mod, name, wrapper)
    return wrapper


def pytest_configure(config):
    import importlib

    import embedview  # the unmodified reference (baseline/_ref)

    # submodules by import path: the package attribute ``embedview.knn`` is the function
    ev_knn, ev_proj, ev_som, ev_gm, ev_engine, ev_cli = (
        importlib.import_module(f"embedview.{m}") for m in ("knn", "projection", "som", "graphmodel", "engine", "cli"))

    import paper_2201_00701_b200 as esom
    from paper_2201_00701_b200 import _lib

    esom.install(embedview, fast=os.environ.get("ESOM_DROPIN_FAST") == "1")
    # count the patched entry points the reference's tests reach (wrappers are
    # installed on the reference's module attributes, after install())
    for mod, names in ((ev_knn, ("knn", "knn_base", "knn_bitonic")),
                       (ev_proj, ("embed", "project_neighbors", "project_point", "scores")),
                       (ev_som, ("som_tick", "quantization_error", "fit_hi_for_new_landmark")),
                       (ev_gm, ("kmeans_tick", "build_knn_graph", "layout_tick"))):
        for name in names:
            w = _counting(mod, name)
            if name in ("knn_base", "knn_bitonic"):
                mod._BACKENDS[name.split("_")[1]] = w
            if name == "embed":  # the by-name importers (ref: engine.py:28, cli.py:15)
                ev_engine.embed = w
                ev_cli.embed = w
    _state["launch0"] = _lib.load().esom_launch_count()
    _state["lib"] = _lib.load()


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("ESOM_DROPIN_REPORT")
    if not path or "lib" not in _state:
        return
    rep = {
        "exitstatus": int(exitstatus),
        "launches": int(_state["lib"].esom_launch_count() - _state["launch0"]),
        "calls": dict(_calls),
        "passed": session.testscollected - session.testsfailed,
        "failed": session.testsfailed,
        "collected": session.testscollected,
    }
    with open(path, "w") as f:
        json.dump(rep, f, indent=1)
