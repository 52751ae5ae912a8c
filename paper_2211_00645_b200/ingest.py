"""Stack ingest straight into page-locked memory.

Reads the reference's recorded-stack formats (ss/source.py:321-474):

* raw: concatenated little-endian uint16 frames, with a JSON sidecar ``<stem>.json``
  holding ``geometry`` (the six SheetGeometry fields), ``timing`` and ``frames``
  (ss/source.py:321-385);
* multi-page 16-bit grayscale TIFF with the same sidecar (ss/source.py:388-395, 450-474).

Where the reference materialises a Python list of per-frame copies
(``_load_raw_frames``, ss/source.py:431-447), raw files are read with one
``readinto`` into a pinned ``(n, H, W)`` buffer, ready for the asynchronous H2D
copies of ``stream.StackStreamer``.  Channel crops (ss/pipeline.py:105-112) are
strided views of the device stack (``channel_views``): ``ssb_deskew`` takes row
and frame strides, so no per-channel copy is made.  Errors are the reference's
``MetadataError`` with the same messages.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

from .errors import MetadataError
from .geometry import SheetGeometry

_GEOMETRY_FIELDS = ("alpha_deg", "scan_step_um", "pixel_pitch_um", "slice_count", "frame_width_px",
                    "frame_height_px")
_TIMING_FIELDS = ("exposure_ms", "readout_ms")


def sidecar_path(path) -> str:
    return os.path.splitext(str(path))[0] + ".json"


def read_sidecar(path):
    """(SheetGeometry, timing dict, frames or None) -- ss/source.py:343-374."""
    sp = sidecar_path(path)
    if not os.path.exists(sp):
        raise MetadataError(f"no sidecar file {sp}")
    with open(sp) as fh:
        try:
            data = json.load(fh)
        except json.JSONDecodeError as exc:
            raise MetadataError(f"sidecar {sp} is not valid JSON: {exc}") from exc
    for section, fields in (("geometry", _GEOMETRY_FIELDS), ("timing", _TIMING_FIELDS)):
        if section not in data:
            raise MetadataError(f"sidecar missing section '{section}'")
        for f in fields:
            if f not in data[section]:
                raise MetadataError(f"sidecar missing field '{section}.{f}'")
    g = data["geometry"]
    geom = SheetGeometry(alpha_deg=g["alpha_deg"], scan_step_um=g["scan_step_um"],
                         pixel_pitch_um=g["pixel_pitch_um"], slice_count=int(g["slice_count"]),
                         frame_width_px=int(g["frame_width_px"]), frame_height_px=int(g["frame_height_px"]))
    t = data["timing"]
    timing = {"exposure_ms": t["exposure_ms"], "readout_ms": t["readout_ms"],
              "trigger_mode": t.get("trigger_mode", "internal")}
    frames = data.get("frames")
    return geom, timing, None if frames is None else int(frames)


def _alloc(n: int, h: int, w: int, pinned: bool, out=None) -> np.ndarray:
    if out is not None:
        if out.dtype != np.uint16 or out.shape != (n, h, w) or not out.flags.c_contiguous:
            raise MetadataError(f"out buffer must be a C-contiguous ({n}, {h}, {w}) uint16 array")
        return out
    if pinned:
        from .stream import pinned_stack

        return pinned_stack(n, h, w)
    return np.empty((n, h, w), dtype=np.uint16)


def _read_parallel(path, view: memoryview, size: int, threads: int = 8, piece: int = 32 << 20) -> None:
    """Read ``size`` bytes of ``path`` into ``view`` with positioned reads on a few threads
    (os.preadv releases the GIL; one thread copying out of the page cache tops out near
    1.6 GB/s on the GPU hosts, several run in parallel)."""
    from concurrent.futures import ThreadPoolExecutor

    fd = os.open(path, os.O_RDONLY)
    try:
        def work(off: int) -> None:
            end = min(size, off + piece)
            while off < end:
                k = os.preadv(fd, [view[off:end]], off)
                if k <= 0:
                    raise MetadataError(f"short read from {path}")
                off += k

        with ThreadPoolExecutor(max_workers=max(1, min(threads, (size + piece - 1) // piece))) as ex:
            list(ex.map(work, range(0, size, piece)))
    finally:
        os.close(fd)


def _load_raw(path, geom: SheetGeometry, count, pinned: bool, out=None) -> np.ndarray:
    w, h = geom.frame_width_px, geom.frame_height_px
    frame_px = w * h
    px = os.path.getsize(path) // 2  # np.fromfile ignores a trailing odd byte (ss/source.py:434)
    if px == 0 or px % frame_px != 0:
        raise MetadataError(f"raw file holds {px} pixels, not a multiple of the sidecar frame size {w}x{h}")
    n = px // frame_px
    if count is not None and n != count:
        raise MetadataError(f"raw file holds {n} frames, sidecar says {count}")
    out = _alloc(n, h, w, pinned, out)
    _read_parallel(path, memoryview(out.reshape(-1).view(np.uint8)), 2 * px)
    if sys.byteorder == "big":  # the file is little-endian ("<u2", ss/source.py:384)
        out.byteswap(inplace=True)
    return out


def _load_tiff(path, geom: SheetGeometry, count, pinned: bool, out=None) -> np.ndarray:
    from PIL import Image

    w, h = geom.frame_width_px, geom.frame_height_px
    # the reference's order of faults (ss/source.py:448-474): any page's pixel type while reading,
    # then page shapes, then the page count
    shape_fault = None
    try:
        with Image.open(path) as im:
            n = getattr(im, "n_frames", 1)
            if out is not None and count is not None and n != count:  # a caller buffer sized by the sidecar
                raise MetadataError(f"TIFF holds {n} pages, sidecar says {count}")
            out = _alloc(n, h, w, pinned, out)
            for i in range(n):
                im.seek(i)
                arr = np.asarray(im)
                if arr.dtype.itemsize != 2 or arr.ndim != 2:
                    raise MetadataError(f"page {i} is not 16-bit grayscale ({arr.dtype}, {arr.ndim}-D)")
                if arr.shape != (h, w):
                    if shape_fault is None:
                        shape_fault = f"TIFF page {i} is {arr.shape[1]}x{arr.shape[0]}, sidecar says {w}x{h}"
                    continue
                out[i] = arr
    except (OSError, SyntaxError) as exc:
        raise MetadataError(f"cannot read TIFF {path}: {exc}") from exc
    if shape_fault is not None:
        raise MetadataError(shape_fault)
    if count is not None and n != count:
        raise MetadataError(f"TIFF holds {n} pages, sidecar says {count}")
    return out


def load_stack(path, geom: SheetGeometry | None = None, *, pinned: bool = True, out=None):
    """Read a recorded stack -> ((n, H, W) uint16 array, geometry, timing dict).

    ``pinned=True`` (default) returns page-locked memory for the H2D pipeline
    (needs a CUDA device); flags beat sidecar as in ``open_stack`` (ss/source.py:477-496).
    ``out``: an existing (n, H, W) uint16 buffer to read into (e.g. a reused
    ``stream.pinned_stack``) -- page-locking a fresh buffer costs more than the read.
    """
    path = str(path)
    if not os.path.exists(path):
        raise MetadataError(f"no such stack file: {path}")
    side_geom, timing, count = None, None, None
    if geom is None:
        side_geom, timing, count = read_sidecar(path)
    elif os.path.exists(sidecar_path(path)):
        _, timing, count = read_sidecar(path)
    geom = geom if geom is not None else side_geom
    if path.lower().endswith((".tif", ".tiff")):
        stack = _load_tiff(path, geom, count, pinned, out)
    else:
        stack = _load_raw(path, geom, count, pinned, out)
    return stack, geom, timing


def channel_views(stack_dev, layout) -> dict:
    """Per-channel crops of a device stack as strided views (no copies).

    ``layout`` is a ``pipeline.ChannelLayout``; returns {channel_id: (n, h, w) view}.
    Mirrors split_channels (ss/pipeline.py:105-112), which copies every crop.
    """
    n, H, W = (int(v) for v in stack_dev.shape)
    layout.validate_frame(W, H)
    return {r.channel_id: stack_dev[:, r.y0:r.y0 + r.height, r.x0:r.x0 + r.width] for r in layout.regions}
