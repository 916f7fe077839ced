"""Install the GPU path into an existing ``tomoplan`` (the reference package).

    import tomoplan
    from paper_2403_07631_b200 import compat
    compat.install(tomoplan)      # tomoplan.build_tomogram & co. now run on the B200

Replaces the hot-path entry points everywhere the reference binds them:
the package namespace (tomoplan/__init__.py:14-45), the defining modules
(tomogram.py, traversability.py, simplify.py, cloud_io.py) and the modules that imported
them by name (cli.py:20, bench.py:19).  Everything downstream (planner,
trajectory, LGA save/load, CLI) consumes the returned objects by duck
typing: ``Tomogram.slices[k].ground/ceiling/cost.values`` are (rows, cols)
float32 numpy arrays, ``ground_stack()`` / ``cost_stack()`` exist.
``uninstall()`` restores the originals.
"""

from __future__ import annotations

import importlib

from . import archive as _arch
from . import cloud_io as _cio
from . import trajectory as _traj
from . import simplify as _simp
from . import tomogram as _tomo
from . import traversability as _trav

# name -> replacement
REPLACEMENTS = {
    "build_tomogram": _tomo.build_tomogram,
    "evaluate_tomogram": _trav.evaluate_tomogram,
    "evaluate_slice": _trav.evaluate_slice,
    "interval_cost": _trav.interval_cost,
    "ground_cost": _trav.ground_cost,
    "slope_magnitudes": _trav.slope_magnitudes,
    "gentle_fraction": _trav.gentle_fraction,
    "terrain_cost_values": _trav.terrain_cost_values,
    "fuse_costs": _trav.fuse_costs,
    "inflate": _trav.inflate,
    "simplify_tomogram": _simp.simplify_tomogram,
    "unique_cells": _simp.unique_cells,
    "save_tomogram": _arch.save_tomogram,   # byte-identical LGA writer (§8 f)
    "load_tomogram": _arch.load_tomogram,
    # load_cloud: a per-install dispatcher (binary PCD straight to HBM, §8 f;
    # the text formats stay with the reference's own parsers), see install()
    "_inflate_ceiling": _traj.inflate_ceiling,  # trajectory.py:277-317 (§8 f)
}

MODULES = ("", ".tomogram", ".traversability", ".simplify", ".cloud_io", ".trajectory", ".cli",
           ".bench")

_saved: list = []


def install(package=None) -> list:
    """Patch ``package`` (default: ``import tomoplan``); returns the patched
    (module, name) pairs."""
    pkg = package if package is not None else importlib.import_module("tomoplan")
    patched = []
    repl = dict(REPLACEMENTS)
    try:
        ref_cio = importlib.import_module(pkg.__name__ + ".cloud_io")
        repl["load_cloud"] = _load_cloud_dispatch(getattr(ref_cio, "load_cloud"))
    except Exception:
        pass
    for suffix in MODULES:
        try:
            mod = importlib.import_module(pkg.__name__ + suffix) if suffix else pkg
        except Exception:  # e.g. bench needs matplotlib
            continue
        for name, fn in repl.items():
            if hasattr(mod, name) and getattr(mod, name) is not fn:
                _saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, fn)
                patched.append((mod.__name__, name))
    return patched


def _load_cloud_dispatch(ref_load_cloud):
    """``load_cloud`` for the patched package: ``pcd_binary`` goes through
    the device ingest (this package), every other format through the
    reference's own parser (cloud_io.py:281-288), saved at install time."""
    if getattr(ref_load_cloud, "_pct_dispatch", False):  # installed twice
        return ref_load_cloud

    def load_cloud(path, fmt):
        if fmt == "pcd_binary":
            return _cio.load_cloud(path, fmt)
        return ref_load_cloud(path, fmt)

    load_cloud.__doc__ = ref_load_cloud.__doc__
    load_cloud._pct_dispatch = True
    return load_cloud


def uninstall() -> None:
    while _saved:
        mod, name, orig = _saved.pop()
        setattr(mod, name, orig)
