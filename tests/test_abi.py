"""CPU-side checks of the C-ABI library: it loads and exports every symbol the
header declares (no compute calls without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "sfft_b200.h")).read()
    return sorted(set(re.findall(r"\b(sfft_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    from paper_2012_08238_b200 import _lib
    h = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert syms, "header declares no symbols"
    for s in syms:
        assert hasattr(h, s), f"missing export {s}"
    assert set(syms) == set(_lib.exported_symbols()), "ctypes table and header disagree"


def test_version_and_error_string():
    from paper_2012_08238_b200 import _lib
    L = _lib.lib()
    assert L.sfft_version() >= 1
    # an argument error is reported without touching the device
    rc = L.sfft_flat_bucketize(7, None, 16, 16, None, 4, 4, 1, None, None, None, None, None,
                               None, None, None, 0, None)
    assert rc == -2
    assert b"dtype" in L.sfft_last_error()
