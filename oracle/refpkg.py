"""Locate and import the REAL reference package ``psdcone`` (test
infrastructure only — never imported by the product package).

Search order: ``oracle/_ref`` (the offline pip install made by
``oracle/make_ref.sh``; it travels to the GPU box with the snapshot), then
``/root/reference/pkg/src`` (the read-only mount in the build container).
Returns ``None`` when neither exists.
"""

from __future__ import annotations

import importlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CANDIDATES = (os.path.join(HERE, "_ref"), "/root/reference/pkg/src")


def location():
    for path in CANDIDATES:
        if os.path.isfile(os.path.join(path, "psdcone", "__init__.py")):
            return path
    return None


def import_psdcone():
    """The reference module, imported from the first candidate that holds it."""
    path = location()
    if path is None:
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    mod = importlib.import_module("psdcone")
    for sub in ("projection", "sketch", "symmetric", "sdls", "experiments", "errors", "bounds"):
        importlib.import_module(f"psdcone.{sub}")
    return mod
