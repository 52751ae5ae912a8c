"""Drop-in for the hot-path half of ``skewstream.pipeline`` on B200.

Same names, signatures, attributes, exception classes and messages as the
reference (ss/pipeline.py:29-112 frame contract, :225-403 projection canvas,
:406-487 warp + emission); the canvas pixels live in HBM and every placement,
band recompute and warp is a hand-written sm_100a kernel from ``libssb.so``.
There is no CPU fallback: without a CUDA device the compute methods raise.

Host views: ``max_pixels`` / ``contributor`` return host numpy copies of the
device canvas (synchronising the canvas stream), so code that reads them the
way the reference's tests and ``LivePipeline`` do keeps working; the device
tensors are ``max_pixels_device`` / ``contributor_device``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib, geometry
from .deskew import canvas_rows_for, deskew_device, require_cuda
from .errors import CapacityError, ParameterError, ProtocolError
from .geometry import SheetGeometry, ViewTransform


# ---------------------------------------------------------------------------
# frames and channel splitting (ss/pipeline.py:29-112)


@dataclass(frozen=True)
class RawFrame:
    """One camera exposure or one channel's crop of it (ss/pipeline.py:34-61)."""

    pixels: np.ndarray
    slice_index: int
    sweep_index: int = 0
    channel_id: int = 0
    timestamp_ns: int = 0

    def __post_init__(self):
        if self.pixels.ndim != 2:
            raise ParameterError("frame pixels must be 2-D (height, width)")
        if self.pixels.dtype != np.uint16:
            raise ParameterError(f"frame pixels must be uint16, got {self.pixels.dtype}")
        if self.slice_index < 0:
            raise ParameterError("slice_index must be >= 0")

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def width(self) -> int:
        return self.pixels.shape[1]


@dataclass(frozen=True)
class ChannelRegion:
    channel_id: int
    x0: int
    y0: int
    width: int
    height: int


@dataclass(frozen=True)
class ChannelLayout:
    """Non-overlapping camera rectangles, one per colour channel (ss/pipeline.py:74-102)."""

    regions: tuple

    def __post_init__(self):
        if not self.regions:
            raise ParameterError("layout needs at least one region")
        for r in self.regions:
            if r.width < 1 or r.height < 1 or r.x0 < 0 or r.y0 < 0:
                raise ParameterError(f"bad region geometry for channel {r.channel_id}")
        for k, a in enumerate(self.regions):
            for b in self.regions[k + 1:]:
                overlap_x = a.x0 < b.x0 + b.width and b.x0 < a.x0 + a.width
                overlap_y = a.y0 < b.y0 + b.height and b.y0 < a.y0 + a.height
                if overlap_x and overlap_y:
                    raise ParameterError(f"regions for channels {a.channel_id} and {b.channel_id} overlap")

    @classmethod
    def full_frame(cls, width: int, height: int, channel_id: int = 0) -> "ChannelLayout":
        return cls(regions=(ChannelRegion(channel_id, 0, 0, width, height),))

    def validate_frame(self, width: int, height: int) -> None:
        for r in self.regions:
            if r.x0 + r.width > width or r.y0 + r.height > height:
                raise ParameterError(f"region for channel {r.channel_id} exceeds {width}x{height} frame")


def split_channels(frame: RawFrame, layout: ChannelLayout) -> list:
    """Per-channel crops as independent copies (ss/pipeline.py:105-112)."""
    layout.validate_frame(frame.width, frame.height)
    return [replace(frame, pixels=frame.pixels[r.y0:r.y0 + r.height, r.x0:r.x0 + r.width].copy(),
                    channel_id=r.channel_id) for r in layout.regions]


# ---------------------------------------------------------------------------
# projection canvas (ss/pipeline.py:239-403)


def _vp(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class _HostView(np.ndarray):
    """Host copy of a device canvas buffer (``max_pixels`` / ``contributor``).

    The reference's canvas buffers are plain mutable arrays (ss/pipeline.py:267-270).  Writes into
    this copy or any view of it -- item assignment or a ufunc with ``out=`` -- mark the owning
    canvas dirty, and its next device operation uploads the host copy first, so an in-place caller
    write is never dropped.  Copies (``.copy()``, ``np.array``) are independent, as in numpy.
    """

    def __array_finalize__(self, obj):
        # views share the owner; fresh arrays (copies) do not
        self._owner = getattr(obj, "_owner", None) if self.base is not None else None

    def _touch(self):
        if self._owner is not None:
            self._owner._host_dirty = True

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._touch()

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kwargs):
        args = [x.view(np.ndarray) if isinstance(x, _HostView) else x for x in inputs]
        if out is not None:
            kwargs["out"] = tuple(o.view(np.ndarray) if isinstance(o, _HostView) else o for o in out)
        res = getattr(ufunc, method)(*args, **kwargs)
        for o in out or ():
            if isinstance(o, _HostView):
                o._touch()
        return res


def _host_view(t: torch.Tensor, owner) -> "_HostView":
    v = t.cpu().numpy().view(_HostView)
    v._owner = owner
    return v


class ProjectionCanvas:
    """Enlarged max-projection canvas of one channel, resident in HBM.

    Global mode max-accumulates a sweep and emits once per stack; rolling mode
    keeps the N most recent slices in a device ring plus a contributor map and
    recomputes only the band a replaced slice touches (ss/pipeline.py:239-247).
    One canvas is owned by one worker; its kernels run on its own CUDA stream.
    """

    def __init__(self, geom: SheetGeometry, shear_px: float, interp: str = "linear",
                 mode: str = "global", max_pixels: int = geometry.DEFAULT_CANVAS_LIMIT_PX):
        if interp not in ("nearest", "linear"):
            raise ParameterError(f"interp must be nearest or linear, got {interp!r}")
        if mode not in ("global", "rolling"):
            raise ParameterError(f"mode must be global or rolling, got {mode!r}")
        self.geom = geom
        self.shear_px = float(shear_px)
        self.interp = interp
        self.mode = mode
        self._pixel_limit = max_pixels
        self.width, self.height = geometry.output_extent(geom, shear_px, max_pixels)
        self._device = require_cuda()
        self.stream = torch.cuda.Stream(self._device)
        self._alloc_canvas()
        self._placed = [False] * geom.slice_count
        self._ring: list = [None] * geom.slice_count
        self._ring_dev = None      # (N, H, W) uint16, allocated on first rolling use
        self._present_dev = None   # (N,) uint8
        self._roll_ws = None       # device list of voxels to re-max (incremental rolling updates)
        self._host_cache = None
        self._host_dirty = False
        self._pending_uploads: list = []  # (copy-done event, pinned host buffer) still being read
        self._staging = None              # pinned two-slot ring for pageable frames: (buffer, event)
        self._stage_next = 0
        self._stage_pending = None
        # True while canvas + contributor equal the full re-max over the ring, so a
        # rolling_replace can take the O(band) incremental path (see ssb_rolling_band)
        self._exact = True
        self._canvas_zero = True

    # -- device buffers ------------------------------------------------------
    def _alloc_canvas(self) -> None:
        with torch.cuda.stream(self.stream):
            self.max_pixels_device = torch.zeros((self.height, self.width), dtype=torch.uint16,
                                                 device=self._device)
            self.contributor_device = torch.full((self.height, self.width), -1, dtype=torch.int16,
                                                 device=self._device)
        self._host_cache = None
        self._canvas_zero = True

    def _ring_empty(self) -> bool:
        return all(rf is None for rf in self._ring)

    def _upload(self, pixels: np.ndarray) -> torch.Tensor:
        """Frame -> device on the canvas stream, asynchronously.  Page-locked frames (e.g. views of
        ``ingest.load_stack`` / ``stream.pinned_stack``) are copied directly; pageable frames are
        first copied (multi-threaded) into a two-slot pinned staging ring, so the H2D copy of one
        frame overlaps the host copy of the next instead of going through the driver's bounce
        buffer synchronously."""
        host = torch.from_numpy(np.ascontiguousarray(pixels))
        if not host.is_pinned():
            host = self._stage(host)
        with torch.cuda.stream(self.stream):
            dev = host.to(self._device, non_blocking=True).unsqueeze(0)
        # RawFrame pixels are immutable (ss/pipeline.py:37-39), so the copy may still be
        # reading them after place() returns: hold the host buffer until its copy completes
        self._hold_until_copied(host)
        return dev

    def _stage(self, host: torch.Tensor) -> torch.Tensor:
        """Copy a pageable frame into the next free slot of the pinned staging ring."""
        ring = self._staging
        if ring is None or tuple(ring[0][0].shape) != tuple(host.shape):
            ring = self._staging = [(torch.empty(tuple(host.shape), dtype=host.dtype, pin_memory=True), None)
                                    for _ in range(2)]
        k = self._stage_next
        self._stage_next ^= 1
        buf, done = ring[k]
        if done is not None:
            done.synchronize()  # the H2D copy that last read this slot has finished
        buf.copy_(host)
        self._stage_pending = k  # _hold_until_copied attaches the slot's copy-done event
        return buf

    def _hold_until_copied(self, host: torch.Tensor) -> None:
        """Keep a pinned host buffer alive until the asynchronous H2D copy just queued on the
        canvas stream has read it (the caller may drop the frame as soon as place() returns)."""
        done = torch.cuda.Event()
        done.record(self.stream)
        if self._stage_pending is not None:  # a staging slot: free again once this copy is done
            k = self._stage_pending
            self._staging[k] = (self._staging[k][0], done)
            self._stage_pending = None
            return
        pending = [(e, h) for e, h in self._pending_uploads if not e.query()]
        pending.append((done, host))
        self._pending_uploads = pending

    @property
    def max_pixels(self) -> np.ndarray:
        """Host copy of the canvas (ss/pipeline.py:267); in-place writes reach the device canvas
        before its next operation (``_HostView``)."""
        if self._host_cache is None:
            self.stream.synchronize()
            self._host_cache = (_host_view(self.max_pixels_device, self), _host_view(self.contributor_device, self))
            self._host_dirty = False
        return self._host_cache[0]

    def _flush_host_writes(self) -> None:
        """Upload host copies that a caller wrote into (see ``_HostView``) before a device op."""
        if not self._host_dirty or self._host_cache is None:
            return
        mp, ct = self._host_cache
        with torch.cuda.stream(self.stream):
            self.max_pixels_device.copy_(torch.from_numpy(np.ascontiguousarray(mp.view(np.ndarray))))
            self.contributor_device.copy_(torch.from_numpy(np.ascontiguousarray(ct.view(np.ndarray))))
        self.stream.synchronize()  # the host arrays may be written again right away
        self._host_dirty = False
        self._exact = self._canvas_zero = False

    @max_pixels.setter
    def max_pixels(self, value) -> None:
        arr = np.ascontiguousarray(value, dtype=np.uint16)
        self.height, self.width = arr.shape
        self._flush_host_writes()  # the other buffer's pending host writes
        with torch.cuda.stream(self.stream):
            self.max_pixels_device = torch.from_numpy(arr).to(self._device)
        self._host_cache = None
        self._exact = self._canvas_zero = False

    @property
    def contributor(self) -> np.ndarray:
        """Host copy of the rolling contributor map (ss/pipeline.py:270)."""
        self.max_pixels  # refresh both host views together
        return self._host_cache[1]

    @contributor.setter
    def contributor(self, value) -> None:
        arr = np.ascontiguousarray(value, dtype=np.int16)
        self._flush_host_writes()
        with torch.cuda.stream(self.stream):
            self.contributor_device = torch.from_numpy(arr).to(self._device)
        self._host_cache = None
        self._exact = self._canvas_zero = False

    @property
    def ring(self) -> list:
        return self._ring

    @ring.setter
    def ring(self, frames) -> None:
        """LivePipeline swaps the ring on a mode change (ss/pipeline.py:864)."""
        self._ring = list(frames)
        self._exact = self._canvas_zero and self._ring_empty()
        if self._present_dev is not None:
            with torch.cuda.stream(self.stream):
                self._present_dev.zero_()
        # the device ring mirrors the assigned frames (allocated by the first store), so a rolling
        # replace_all right after the assignment re-maxes from resident frames
        for rf in self._ring:
            if rf is not None:
                self._ring_store(rf)

    # -- placement grid --------------------------------------------------------
    def row_span(self, slice_index: int) -> tuple[int, int]:
        """Inclusive canvas rows of a slice (ss/pipeline.py:274-281)."""
        return geometry.row_span(slice_index, self.shear_px, self.geom.frame_height_px, self.interp)

    def _check_frame(self, frame: RawFrame) -> None:
        """Same checks and messages as ss/pipeline.py:292-312."""
        if frame.width != self.width:
            raise ParameterError(f"frame width {frame.width} does not match canvas width {self.width}")
        if frame.height != self.geom.frame_height_px:
            raise ParameterError(
                f"frame height {frame.height} does not match geometry {self.geom.frame_height_px}")
        if frame.slice_index >= self.geom.slice_count:
            raise ParameterError(
                f"slice_index {frame.slice_index} out of range (stack of {self.geom.slice_count})")
        lo, hi = self.row_span(frame.slice_index)
        if lo < 0 or hi >= self.height:
            raise CapacityError(
                f"slice {frame.slice_index} spans rows {lo}..{hi} on a {self.height}-row canvas; "
                "canvas was mis-sized")

    # -- global mode -------------------------------------------------------------
    def place(self, frame: RawFrame) -> tuple[int, int]:
        """Max-accumulate one slice into the device canvas (ss/pipeline.py:316-323)."""
        self._check_frame(frame)
        self._flush_host_writes()
        lo, hi = self.row_span(frame.slice_index)
        raw = self._upload(frame.pixels)
        # one fused launch over the slice's band: rows lo..hi, XY folded in place
        deskew_device(raw, self.shear_px, self.interp, first_slice=frame.slice_index,
                      canvas_rows=self.height, u_begin=lo, u_count=hi - lo + 1,
                      projection_axes=(0,), write_volume=False,
                      projections={0: self.max_pixels_device[lo:hi + 1]}, xy_accumulate=True,
                      stream=self.stream)
        self._placed[frame.slice_index] = True
        self._host_cache = None
        self._exact = self._canvas_zero = False
        return lo, hi

    def place_stack(self, frames: torch.Tensor, first_slice: int = 0) -> None:
        """Place n consecutive device-resident slices in one fused launch."""
        self._flush_host_writes()
        n = int(frames.shape[0])
        if first_slice < 0 or first_slice + n > self.geom.slice_count:
            raise ParameterError("slice range out of range")
        deskew_device(frames, self.shear_px, self.interp, first_slice=first_slice,
                      canvas_rows=self.height, projection_axes=(0,), write_volume=False,
                      projections={0: self.max_pixels_device}, xy_accumulate=True, stream=self.stream)
        for i in range(first_slice, first_slice + n):
            self._placed[i] = True
        self._host_cache = None
        self._exact = self._canvas_zero = False

    @property
    def placed_count(self) -> int:
        return sum(self._placed)

    def finalize_global(self) -> np.ndarray:
        """Emit the finished projection and reset (ss/pipeline.py:329-336)."""
        if not all(self._placed):
            missing = self._placed.count(False)
            raise ProtocolError(f"finalize with {missing} slice(s) not yet placed")
        out = self.max_pixels.copy()
        self.reset()
        return out

    def finalize_global_device(self) -> torch.Tensor:
        """Device variant: returns a device copy without a host sync."""
        self._flush_host_writes()
        if not all(self._placed):
            raise ProtocolError(f"finalize with {self._placed.count(False)} slice(s) not yet placed")
        with torch.cuda.stream(self.stream):
            out = self.max_pixels_device.clone()
        self.reset()
        return out

    def reset(self) -> None:
        self._flush_host_writes()
        with torch.cuda.stream(self.stream):
            self.max_pixels_device.zero_()
            self.contributor_device.fill_(-1)
        self._placed = [False] * self.geom.slice_count
        self._host_cache = None
        self._canvas_zero = True
        self._exact = self._ring_empty()

    # -- rolling mode --------------------------------------------------------------
    def _ring_store(self, frame: RawFrame) -> None:
        n, h, w = self.geom.slice_count, self.geom.frame_height_px, frame.width
        with torch.cuda.stream(self.stream):
            if self._ring_dev is None or tuple(self._ring_dev.shape) != (n, h, w):
                self._ring_dev = torch.zeros((n, h, w), dtype=torch.uint16, device=self._device)
                self._present_dev = torch.zeros((n,), dtype=torch.uint8, device=self._device)
            host = torch.from_numpy(np.ascontiguousarray(frame.pixels))
            if not host.is_pinned():
                host = self._stage(host)  # pageable: through the pinned staging ring (see _upload)
            self._ring_dev[frame.slice_index].copy_(host, non_blocking=True)
            self._present_dev[frame.slice_index] = 1
        self._hold_until_copied(host)  # the async copy may still read it

    def rolling_replace(self, frame: RawFrame) -> tuple[int, int]:
        """Swap in the newest version of a slice and refresh its band (ss/pipeline.py:345-359)."""
        self._flush_host_writes()
        if self.mode != "rolling":
            raise ProtocolError("rolling_replace on a canvas in global mode")
        self._check_frame(frame)
        self._ring[frame.slice_index] = frame
        self._ring_store(frame)
        lo, hi = self.row_span(frame.slice_index)
        self._recompute_band(lo, hi, frame.slice_index if self._exact else -1)
        return lo, hi

    def _recompute_band(self, lo: int, hi: int, replaced: int = -1) -> None:
        """ss/pipeline.py:361-377 on device (strict '>' max, first-max-wins contributor).

        replaced >= 0 takes the incremental path: exact while the canvas equals the
        full ring re-max (``_exact``); otherwise the whole band is re-maxed.
        """
        lib = _lib.load()
        if self._ring_dev is None:  # nothing stored yet: an all-absent ring of the right shape
            with torch.cuda.stream(self.stream):
                self._ring_dev = torch.zeros((self.geom.slice_count, self.geom.frame_height_px, self.width),
                                             dtype=torch.uint16, device=self._device)
                self._present_dev = torch.zeros((self.geom.slice_count,), dtype=torch.uint8, device=self._device)
        ws, ws_bytes = None, 0
        if replaced >= 0:
            ws_bytes = int(lib.ssb_rolling_workspace_bytes(hi - lo + 1, self.width))
            if self._roll_ws is None or self._roll_ws.numel() < ws_bytes:
                with torch.cuda.stream(self.stream):
                    self._roll_ws = torch.empty(ws_bytes, dtype=torch.uint8, device=self._device)
            ws = self._roll_ws
        _lib.check(lib.ssb_rolling_band(
            _vp(self._ring_dev), _vp(self._present_dev), self.geom.slice_count,
            self.geom.frame_height_px, self.width, self.shear_px, _lib.INTERP[self.interp], lo, hi,
            _vp(self.max_pixels_device), _vp(self.contributor_device), self.height, replaced,
            _vp(ws), ws_bytes, ctypes.c_void_p(self.stream.cuda_stream)))
        self._host_cache = None
        self._canvas_zero = False

    def replace_all(self, shear_px: float | None = None) -> None:
        """Rebuild the canvas, optionally under a new shear (ss/pipeline.py:379-398)."""
        if shear_px is not None:
            self.shear_px = float(shear_px)
        self.width, self.height = geometry.output_extent(self.geom, self.shear_px, self._pixel_limit)
        self._alloc_canvas()
        self._placed = [False] * self.geom.slice_count
        # re-adding every live slot in ring order onto a zero canvas with the incremental
        # rule yields the full re-max (ties keep the earliest slot)
        self._exact = True
        if self.mode == "rolling":
            # the ring's frames are already resident: re-add each live slot's band from the
            # device ring (no re-upload), in ring order, with the incremental rule
            for rf in self._ring:
                if rf is not None:
                    self._check_frame(rf)
                    lo, hi = self.row_span(rf.slice_index)
                    self._recompute_band(lo, hi, rf.slice_index)


def deskew_place(canvas: ProjectionCanvas, frame: RawFrame) -> tuple[int, int]:
    """Functional alias of ProjectionCanvas.place (ss/pipeline.py:401-403)."""
    return canvas.place(frame)


# ---------------------------------------------------------------------------
# warp + emission (ss/pipeline.py:406-487)


@dataclass(frozen=True)
class StageTimings:
    """Per-stack stage durations plus output lag (ss/pipeline.py:118-138)."""

    acquisition_ms: float
    processing_ms: float
    plotting_ms: float
    lag_ms: float

    def __post_init__(self):
        for name in ("acquisition_ms", "processing_ms", "plotting_ms", "lag_ms"):
            if getattr(self, name) < 0:
                raise ParameterError(f"{name} must be >= 0")

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("acquisition_ms", "processing_ms", "plotting_ms", "lag_ms")}


@dataclass(frozen=True)
class DisplayImage:
    """One emitted view (ss/pipeline.py:410-431)."""

    pixels: np.ndarray
    channel_id: int
    sweep_index: int
    slice_index: int
    view_angle_deg: float
    mode: str
    out_pitch_um: float
    lateral_pitch_um: float
    timings: object = None
    emitted_at_ns: int = 0

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def width(self) -> int:
        return self.pixels.shape[1]


def warp_projection_device(projection: torch.Tensor, warp_scale: float,
                           stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """1-D fp64 row resample on device (ss/pipeline.py:434-457)."""
    if warp_scale <= 0:
        raise ParameterError(f"warp_scale must be > 0, got {warp_scale}")
    rows, cols = (int(v) for v in projection.shape)
    out_rows = int(round(rows * warp_scale))
    if out_rows < 1:
        raise ParameterError(f"warp of {rows} rows by {warp_scale} leaves no output rows")
    stream = stream or torch.cuda.current_stream(projection.device)
    src = projection.contiguous()
    with torch.cuda.stream(stream):
        out = torch.empty((out_rows, cols), dtype=torch.uint16, device=projection.device)
    lib = _lib.load()
    _lib.check(lib.ssb_warp_rows(_vp(src), rows, cols, float(warp_scale), _vp(out), out_rows,
                                 ctypes.c_void_p(stream.cuda_stream)))
    return out


def warp_projection(projection, warp_scale: float):
    """Drop-in of ss/pipeline.py:434-457: numpy in -> numpy out (torch CUDA in -> CUDA out)."""
    if warp_scale <= 0:
        raise ParameterError(f"warp_scale must be > 0, got {warp_scale}")
    if isinstance(projection, torch.Tensor) and projection.is_cuda:
        return warp_projection_device(projection, warp_scale)
    arr = np.ascontiguousarray(projection, dtype=np.uint16)
    rows = arr.shape[0]
    if int(round(rows * warp_scale)) < 1:
        raise ParameterError(f"warp of {rows} rows by {warp_scale} leaves no output rows")
    dev = require_cuda()
    out = warp_projection_device(torch.from_numpy(arr).to(dev), warp_scale)
    return out.cpu().numpy()


def warp_and_emit(projection, vt: ViewTransform, *, channel_id: int = 0, sweep_index: int = 0,
                  slice_index: int = 0, mode: str = "global", lateral_pitch_um: float | None = None,
                  timings=None, emitted_at_ns: int = 0) -> DisplayImage:
    """Warp a finished projection and tag it for display (ss/pipeline.py:460-487)."""
    pixels = warp_projection(projection, vt.warp_scale)
    return DisplayImage(pixels=pixels, channel_id=channel_id, sweep_index=sweep_index,
                        slice_index=slice_index, view_angle_deg=vt.view_angle_deg, mode=mode,
                        out_pitch_um=vt.out_pitch_um,
                        lateral_pitch_um=vt.out_pitch_um if lateral_pitch_um is None else lateral_pitch_um,
                        timings=timings, emitted_at_ns=emitted_at_ns)
