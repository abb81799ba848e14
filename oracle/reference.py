"""Load the REFERENCE package read-only under the alias ``volmoments_ref`` --
TEST / BASELINE INFRASTRUCTURE ONLY (never imported by the product package).

Where it is found, in order: ``baseline/_ref/volmoments`` (the offline install
the driver keeps beside the repo, ``pip install --target baseline/_ref``; it
travels to the GPU box) and ``/root/reference/pkg/src/volmoments`` (the build
container).  Returns None when neither exists, e.g. a fresh GPU box without
the install: callers report the reference legs as unavailable.
"""
from __future__ import annotations

import importlib.util
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(_ROOT, "baseline", "_ref", "volmoments"), "/root/reference/pkg/src/volmoments")


def location() -> str | None:
    for path in CANDIDATES:
        if os.path.exists(os.path.join(path, "__init__.py")):
            return path
    return None


def load():
    """The reference package as module ``volmoments_ref`` (cached), or None."""
    if "volmoments_ref" in sys.modules:
        return sys.modules["volmoments_ref"]
    path = location()
    if path is None:
        return None
    spec = importlib.util.spec_from_file_location("volmoments_ref", os.path.join(path, "__init__.py"),
                                                  submodule_search_locations=[path])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["volmoments_ref"] = mod
    spec.loader.exec_module(mod)
    return mod
