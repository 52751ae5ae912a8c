"""libssb.so builds, loads without a GPU, and exports every symbol include/ssb.h declares."""

import ctypes
import os
import re

from paper_2211_00645_b200 import _build, _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(REPO, "include", "ssb.h")).read()
    return sorted(set(re.findall(r"\b(ssb_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_loads():
    path = _build.build()
    assert os.path.exists(path)
    lib = _lib.load()
    assert lib.ssb_version() == 200


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(_build.build())
    decl = declared_symbols()
    assert set(decl) == set(_lib.EXPORTS), "python binding list out of sync with the header"
    for name in decl:
        assert hasattr(lib, name), name


def test_workspace_query_and_validation_without_gpu():
    lib = _lib.load()
    d = _lib.DeskewDesc(n=512, height=2048, width=2048, first_slice=0, shear_px=0.8660254037844386,
                        interp=1, formula=0, u_begin=0, u_count=2491, reduce=0, flags=0)
    assert lib.ssb_deskew_workspace_bytes(ctypes.byref(d)) > 0
    bad = _lib.DeskewDesc(n=1, height=0, width=4, first_slice=0, shear_px=1.0, interp=1, formula=0,
                          u_begin=0, u_count=2, reduce=0, flags=0)
    rc = lib.ssb_deskew(ctypes.byref(bad), None, None, None, None, None, None, 0, None)
    assert rc == _lib.SSB_ERR_PARAM
    assert b"shape" in lib.ssb_last_error()
    assert lib.ssb_warp_rows(None, 4, 4, 0.0, None, 4, None) == _lib.SSB_ERR_PARAM
    assert lib.ssb_combine(None, None, 4, 1, 16, None) == _lib.SSB_ERR_PARAM
