"""ctypes binding of the C oracle (``deskew_oracle.c``) -- TEST INFRASTRUCTURE ONLY.

Builds ``oracle/build/liboracle.so`` with ``make`` on first use (gcc is present
both here and on the GPU box).  Same semantics as ``deskew_oracle.py``; used for
parity checks at sizes where the numpy oracle is slow.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
_lock = threading.Lock()
_lib = None

INTERP = {"nearest": 0, "linear": 1}
FORMULA = {"canvas": 0, "npinterp": 1}
REDUCE = {"max": 0, "sum": 1}


def build() -> str:
    src = os.path.join(HERE, "deskew_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = ctypes.CDLL(build())
            p, i64, d, i = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
            _lib.oracle_deskew.argtypes = [p, i64, i64, i64, i64, d, i, i, i64, i64, p, p, p, p, i]
            _lib.oracle_deskew.restype = i
            _lib.oracle_warp.argtypes = [p, i64, i64, d, p, i64]
            _lib.oracle_warp.restype = i
        return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def deskew(stack: np.ndarray, shear: float, interp: str = "linear", formula: str = "canvas",
           first_slice: int = 0, u_begin: int = 0, u_count: int | None = None,
           want_volume: bool = True, axes=(0, 1, 2), reduce: str = "max"):
    """Returns (volume or None, {axis: projection}); projections uint16 (max) / uint32 (sum)."""
    from .deskew_oracle import canvas_height

    stack = np.ascontiguousarray(stack, dtype=np.uint16)
    n, h, w = stack.shape
    if u_count is None:
        u_count = canvas_height(first_slice + n, h, shear) - u_begin
    vol = np.empty((n, u_count, w), np.uint16) if want_volume else None
    xy = np.empty((u_count, w), np.uint32) if 0 in axes else None
    xz = np.empty((n, w), np.uint32) if 1 in axes else None
    yz = np.empty((n, u_count), np.uint32) if 2 in axes else None
    rc = lib().oracle_deskew(_ptr(stack), n, h, w, first_slice, float(shear), INTERP[interp],
                             FORMULA[formula], u_begin, u_count, _ptr(vol), _ptr(xy), _ptr(xz),
                             _ptr(yz), REDUCE[reduce])
    if rc != 0:
        raise MemoryError("oracle_deskew failed")
    out = {}
    for ax, arr in ((0, xy), (1, xz), (2, yz)):
        if arr is not None:
            out[ax] = arr.astype(np.uint16) if reduce == "max" else arr
    return vol, out


def warp(proj: np.ndarray, scale: float) -> np.ndarray:
    proj = np.ascontiguousarray(proj, dtype=np.uint16)
    rows, cols = proj.shape
    out_rows = int(round(rows * scale))
    out = np.empty((out_rows, cols), np.uint16)
    lib().oracle_warp(_ptr(proj), rows, cols, float(scale), _ptr(out), out_rows)
    return out
