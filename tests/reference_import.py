"""Locate the reference package for the integration tests: the offline install under
baseline/_ref (travels to the GPU box) or, in the build container, /root/reference."""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def import_reference():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "ensemblegate").is_dir() and str(p) not in sys.path:
            sys.path.append(str(p))
    try:
        return importlib.import_module("ensemblegate")
    except ImportError:
        return None
