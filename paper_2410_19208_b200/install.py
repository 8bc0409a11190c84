"""Rebind the reference ``psdcone`` package onto the B200 path.

The reference binds hot-path names at import time:
``sdls.py:16-18`` (project, ProjectorConfig, min_eig_magnitude,
exact_psd_projection), ``experiments.py:17`` (ran_proj, ran_proj_scal),
``projection.py:10`` (range_finder, min_eig_magnitude).  ``install()``
replaces those module attributes (and the package-level re-exports) with this
package's implementations and points our error registry at psdcone's own
exception classes, so callers that catch ``psdcone.AlphaTooSmall`` keep
working.  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import importlib

from . import errors

_SAVED = {}

# (module, attribute) → our implementation name
_TARGETS = {
    ("psdcone", "project"): "project",
    ("psdcone", "ran_proj"): "ran_proj",
    ("psdcone", "ran_proj_scal"): "ran_proj_scal",
    ("psdcone", "range_finder"): "range_finder",
    ("psdcone", "power_iteration"): "power_iteration",
    ("psdcone", "min_eig_magnitude"): "min_eig_magnitude",
    ("psdcone", "require_symmetric"): "require_symmetric",
    ("psdcone", "eigh"): "eigh",
    ("psdcone", "exact_psd_projection"): "exact_psd_projection",
    ("psdcone.projection", "project"): "project",
    ("psdcone.projection", "ran_proj"): "ran_proj",
    ("psdcone.projection", "ran_proj_scal"): "ran_proj_scal",
    ("psdcone.projection", "range_finder"): "range_finder",
    ("psdcone.projection", "min_eig_magnitude"): "min_eig_magnitude",
    ("psdcone.sketch", "range_finder"): "range_finder",
    ("psdcone.sketch", "power_iteration"): "power_iteration",
    ("psdcone.sketch", "min_eig_magnitude"): "min_eig_magnitude",
    ("psdcone.sdls", "project"): "project",
    ("psdcone.sdls", "min_eig_magnitude"): "min_eig_magnitude",
    ("psdcone.sdls", "exact_psd_projection"): "exact_psd_projection",
    ("psdcone", "solve"): "solve",
    ("psdcone.sdls", "solve"): "solve",
    ("psdcone.experiments", "ran_proj"): "ran_proj",
    ("psdcone.experiments", "ran_proj_scal"): "ran_proj_scal",
    ("psdcone.experiments", "projection_error_sweep"): "projection_error_sweep",
    ("psdcone", "projection_error_sweep"): "projection_error_sweep",
}


def install(psdcone_module=None):
    """Route the reference package's hot path through libpsdproj.so."""
    import paper_2410_19208_b200 as ours

    ref = psdcone_module or importlib.import_module("psdcone")
    ref_errors = importlib.import_module(ref.__name__ + ".errors")
    for name in list(errors.REGISTRY):
        _SAVED.setdefault(("errors", name), errors.REGISTRY[name])
        if hasattr(ref_errors, name):
            errors.REGISTRY[name] = getattr(ref_errors, name)
        else:  # DeviceError has no reference analogue: catchable as psdcone.PsdconeError too
            errors.REGISTRY[name] = type(name, (errors.REGISTRY[name], ref_errors.PsdconeError), {})
    # our ProjectorConfig/RangeParams validation must accept the reference's objects too
    for (modname, attr), impl in _TARGETS.items():
        modname = modname.replace("psdcone", ref.__name__, 1)
        mod = importlib.import_module(modname)
        if hasattr(mod, attr):
            _SAVED.setdefault((modname, attr), getattr(mod, attr))
            setattr(mod, attr, getattr(ours, impl))
    return ref


def original(modname, attr):
    """The reference implementation ``install()`` replaced (e.g. to compare
    against it while installed); ``None`` if that name was not rebound."""
    for (mod, name), val in _SAVED.items():
        if name == attr and mod.split(".", 1)[-1] == modname.split(".", 1)[-1] and mod != "errors":
            return val
    return None


def uninstall():
    for key, val in list(_SAVED.items()):
        modname, attr = key
        if modname == "errors":
            errors.REGISTRY[attr] = val
        else:
            setattr(importlib.import_module(modname), attr, val)
    _SAVED.clear()
