"""ctypes binding of ``libssb.so`` (the C ABI declared in ``include/ssb.h``).

The shared library is built in-tree (``__graft_entry__.build()`` ->
``paper_2211_00645_b200/lib/libssb.so``).  There is no CPU fallback: if the
library or a CUDA device is missing, every compute entry point raises
``DeviceError`` loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CapacityError, DeviceError, ParameterError, ProtocolError, SkewstreamError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libssb.so")

SSB_OK, SSB_ERR_PARAM, SSB_ERR_CAPACITY, SSB_ERR_PROTOCOL, SSB_ERR_CUDA = 0, 1, 2, 3, 4
INTERP = {"nearest": 0, "linear": 1}
FORMULA = {"canvas": 0, "npinterp": 1}
REDUCE = {"max": 0, "sum": 1}
FLAG_XY_ACCUMULATE = 1
FLAG_XY_U32 = 2

#: every symbol include/ssb.h declares (checked by tests/test_abi.py)
EXPORTS = ("ssb_version", "ssb_last_error", "ssb_launch_count", "ssb_profile_enable",
           "ssb_profile_read", "ssb_deskew_workspace_bytes",
           "ssb_deskew", "ssb_deskew_batch_workspace_bytes", "ssb_deskew_batch", "ssb_rolling_workspace_bytes", "ssb_rolling_band", "ssb_warp_rows", "ssb_combine",
           "ssb_encode_gray8_stats_bytes", "ssb_encode_gray8")


class DeskewDesc(ctypes.Structure):
    """Mirror of ``ssb_deskew_desc`` (include/ssb.h)."""

    _fields_ = [
        ("n", ctypes.c_int64),
        ("height", ctypes.c_int64),
        ("width", ctypes.c_int64),
        ("first_slice", ctypes.c_int64),
        ("shear_px", ctypes.c_double),
        ("interp", ctypes.c_int32),
        ("formula", ctypes.c_int32),
        ("u_begin", ctypes.c_int64),
        ("u_count", ctypes.c_int64),
        ("reduce", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("row_stride", ctypes.c_int64),
        ("frame_stride", ctypes.c_int64),
    ]


_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load and type the library once; raise DeviceError if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"native library {path} not built; run __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        p, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        pdesc = ctypes.POINTER(DeskewDesc)
        lib.ssb_version.restype = ctypes.c_int
        lib.ssb_last_error.restype = ctypes.c_char_p
        lib.ssb_launch_count.restype = i64
        lib.ssb_profile_enable.argtypes = [i32]
        lib.ssb_profile_enable.restype = ctypes.c_int
        lib.ssb_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
        lib.ssb_profile_read.restype = ctypes.c_int
        lib.ssb_deskew_workspace_bytes.argtypes = [pdesc]
        lib.ssb_deskew_workspace_bytes.restype = ctypes.c_size_t
        lib.ssb_deskew.argtypes = [pdesc, p, p, p, p, p, p, ctypes.c_size_t, p]
        lib.ssb_deskew.restype = ctypes.c_int
        lib.ssb_deskew_batch_workspace_bytes.argtypes = [pdesc, i64]
        lib.ssb_deskew_batch_workspace_bytes.restype = ctypes.c_size_t
        lib.ssb_deskew_batch.argtypes = [pdesc, i64, p, p, p, p, p, p, ctypes.c_size_t, p]
        lib.ssb_deskew_batch.restype = ctypes.c_int
        lib.ssb_rolling_workspace_bytes.argtypes = [i64, i64]
        lib.ssb_rolling_workspace_bytes.restype = ctypes.c_size_t
        lib.ssb_rolling_band.argtypes = [p, p, i64, i64, i64, d, i32, i64, i64, p, p, i64, i64, p, ctypes.c_size_t, p]
        lib.ssb_rolling_band.restype = ctypes.c_int
        lib.ssb_warp_rows.argtypes = [p, i64, i64, d, p, i64, p]
        lib.ssb_warp_rows.restype = ctypes.c_int
        lib.ssb_combine.argtypes = [p, p, i64, i32, i32, p]
        lib.ssb_combine.restype = ctypes.c_int
        lib.ssb_encode_gray8_stats_bytes.restype = ctypes.c_size_t
        lib.ssb_encode_gray8.argtypes = [p, i64, p, p, ctypes.c_size_t, p]
        lib.ssb_encode_gray8.restype = ctypes.c_int
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a status code onto the reference's exception classes (ss/errors.py)."""
    if rc == SSB_OK:
        return
    msg = (_lib.ssb_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    if rc == SSB_ERR_PARAM:
        raise ParameterError(msg)
    if rc == SSB_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == SSB_ERR_PROTOCOL:
        raise ProtocolError(msg)
    if rc == SSB_ERR_CUDA:
        raise DeviceError(msg)
    raise SkewstreamError(f"libssb status {rc}: {msg}")


def launch_count() -> int:
    return int(load().ssb_launch_count())


def profile_enable(on: bool) -> None:
    check(load().ssb_profile_enable(1 if on else 0))


def profile_read() -> tuple[float, int]:
    """(summed device ms of the timed main kernels, number of launches); clears."""
    ms, n = ctypes.c_double(0.0), ctypes.c_int64(0)
    check(load().ssb_profile_read(ctypes.byref(ms), ctypes.byref(n)))
    return float(ms.value), int(n.value)
