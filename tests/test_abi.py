"""CPU: the C-ABI library loads and exports every entry point include/ensemble_b200.h declares."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

from paper_2003_01538_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "ensemble_b200.h"


def declared() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^(?:int|const char\*)\s+(eb_\w+)\(", text, flags=re.M))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("eb_engine_create", "eb_forward", "eb_add_op", "eb_finalize", "eb_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in sorted(declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert declared() == set(_lib.EXPORTED)


def test_abi_version_and_errors_without_gpu():
    lib = _lib.load()
    assert lib.eb_abi_version() == 1
    # argument validation happens before touching the device
    h = ctypes.c_void_p()
    rc = lib.eb_engine_create(0, 0, 3, 224, 224, ctypes.byref(h))
    assert rc == _lib.EB_E_INVALID
    assert "geometry" in _lib.last_error()
