"""Device-level deskew + projection engine and the additive ``deskew_volume`` API.

``deskew_device`` is the thin Python layer over ``ssb_deskew`` (include/ssb.h):
it validates arguments exactly like the reference does, allocates outputs as
torch CUDA tensors (torch is only the buffer type here) and launches the fused
kernel on the caller's stream.  ``deskew_volume`` is the north_star's
reference-shaped entry point (stack, geometry, shear, interpolation, projection
axes, reduce); host stacks go through the pinned multi-stream H2D pipeline of
``stream.py``.

Index conventions (reference): frames are (H, W) uint16, W contiguous
(ss/pipeline.py:34-61); slice i sits at canvas row offset i*s
(ss/geometry.py:1-22); the volume is (N, U, W) uint16, the reference's pile
layout (ss/phantom.py:390); projection axis 0 = XY (the reference's canvas,
ss/pipeline.py:316-336), 1 = XZ, 2 = YZ.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, ParameterError
from .geometry import _ceil_snapped

_AXES = (0, 1, 2)


@dataclass
class DeskewResult:
    """Outputs of one deskew call.

    volume       (n, u_count, W) uint16 or None
    projections  {axis: array}; max -> uint16, sum -> uint32
    canvas_rows  U of the full canvas; u_begin/u_count the covered row window
    """

    volume: object
    projections: dict = field(default_factory=dict)
    canvas_rows: int = 0
    u_begin: int = 0
    u_count: int = 0

    @property
    def xy(self):
        return self.projections.get(0)

    @property
    def xz(self):
        return self.projections.get(1)

    @property
    def yz(self):
        return self.projections.get(2)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible; this package has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def canvas_rows_for(n_total: int, height: int, shear_px: float) -> int:
    """U = H + ceil((N-1)*s - 1e-9) (ss/geometry.py:141)."""
    return height + _ceil_snapped((n_total - 1) * shear_px)


def check_options(interp: str, reduce: str = "max", formula: str = "canvas", axes=_AXES) -> tuple:
    if interp not in _lib.INTERP:
        raise ParameterError(f"interp must be nearest or linear, got {interp!r}")
    if reduce not in _lib.REDUCE:
        raise ParameterError(f"reduce must be max or sum, got {reduce!r}")
    if formula not in _lib.FORMULA:
        raise ParameterError(f"formula must be canvas or npinterp, got {formula!r}")
    axes = tuple(sorted(set(int(a) for a in axes)))
    if any(a not in _AXES for a in axes):
        raise ParameterError(f"projection axes must be drawn from (0, 1, 2), got {axes}")
    return axes


def proj_dtype(reduce: str) -> torch.dtype:
    return torch.uint16 if reduce == "max" else torch.uint32


def _vp(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class _Workspaces:
    """One growable scratch buffer per CUDA stream (kernels on different streams
    must not share partial-projection scratch), least-recently-used streams evicted beyond
    ``max_streams`` (callers that create streams per call, e.g. one StackStreamer per
    ``deskew_volume``, would otherwise keep a buffer per pooled stream).  An evicted buffer is
    released through torch's caching allocator, which orders its reuse after the work already
    queued on its stream."""

    def __init__(self, max_streams: int = 16):
        from collections import OrderedDict

        self._lock = threading.Lock()
        self._bufs = OrderedDict()
        self.max_streams = max_streams

    def get(self, nbytes: int, stream: torch.cuda.Stream) -> torch.Tensor:
        key = (stream.device.index, stream.cuda_stream)
        with self._lock:
            buf = self._bufs.pop(key, None)
            if buf is None or buf.numel() < nbytes:
                with torch.cuda.stream(stream):
                    buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=stream.device)
            self._bufs[key] = buf  # most recently used last
            while len(self._bufs) > self.max_streams:
                self._bufs.popitem(last=False)
            return buf


_workspaces = _Workspaces()


def make_desc(n, h, w, first_slice, shear_px, interp, formula, u_begin, u_count, reduce,
              xy_accumulate=False, row_stride=0, frame_stride=0, xy_u32=False) -> _lib.DeskewDesc:
    return _lib.DeskewDesc(
        n=n, height=h, width=w, first_slice=first_slice, shear_px=float(shear_px),
        interp=_lib.INTERP[interp], formula=_lib.FORMULA[formula], u_begin=u_begin,
        u_count=u_count, reduce=_lib.REDUCE[reduce],
        flags=(_lib.FLAG_XY_ACCUMULATE if xy_accumulate else 0) | (_lib.FLAG_XY_U32 if xy_u32 else 0),
        row_stride=row_stride, frame_stride=frame_stride,
    )


def deskew_device(raw: torch.Tensor, shear_px: float, interp: str = "linear", *,
                  formula: str = "canvas", first_slice: int = 0, canvas_rows: int | None = None,
                  u_begin: int = 0, u_count: int | None = None, projection_axes=_AXES,
                  reduce: str = "max", write_volume: bool = True, volume: torch.Tensor | None = None,
                  projections: dict | None = None, xy_accumulate: bool = False, xy_u32: bool = False,
                  stream: torch.cuda.Stream | None = None) -> DeskewResult:
    """Fused deskew + projections of device-resident frames (one ``ssb_deskew``).

    raw: CUDA uint16 (n, H, W); frame k is global slice first_slice+k.  Columns must be
    contiguous; rows and frames may be strided (a channel crop of a wider camera frame,
    ss/pipeline.py:105-112, is deskewed in place without a copy).
    Output buffers may be passed in (``volume``, ``projections``) to avoid
    allocation; ``xy_accumulate`` folds into an existing XY (streaming place).  ``xy_u32`` (max
    mode): ``projections[0]`` is a caller-owned int32 (U, W) accumulator, max-folded in place and
    never narrowed (``SSB_FLAG_XY_U32``; the chunked streamer keeps one across its chunks).
    """
    axes = check_options(interp, reduce, formula, projection_axes)
    if not isinstance(raw, torch.Tensor) or not raw.is_cuda:
        raise ParameterError("raw must be a CUDA tensor (use deskew_volume for host stacks)")
    if raw.dtype != torch.uint16:
        raise ParameterError(f"frame pixels must be uint16, got {raw.dtype}")
    if raw.dim() != 3:
        raise ParameterError("raw must be (n, H, W)")
    if raw.shape[2] > 1 and raw.stride(2) != 1:
        raw = raw.contiguous()
    n_, h_, w_ = (int(v) for v in raw.shape)
    row_stride = int(raw.stride(1)) if h_ > 1 else w_
    frame_stride = int(raw.stride(0)) if n_ > 1 else row_stride * h_
    if row_stride < w_ or frame_stride < row_stride * (h_ - 1) + w_:
        raw = raw.contiguous()
        row_stride, frame_stride = w_, w_ * h_
    if shear_px < 0:
        raise ParameterError(f"shear_px must be >= 0, got {shear_px}")
    if first_slice < 0:
        raise ParameterError("first_slice must be >= 0")
    n, h, w = (int(v) for v in raw.shape)
    if canvas_rows is None:
        canvas_rows = canvas_rows_for(first_slice + max(n, 1), h, shear_px)
    if u_count is None:
        u_count = canvas_rows - u_begin
    if u_begin < 0 or u_count < 0:
        raise ParameterError("bad canvas row window")
    dev = raw.device
    stream = stream or torch.cuda.current_stream(dev)
    projections = dict(projections or {})
    pdt = proj_dtype(reduce)
    shapes = {0: (u_count, w), 1: (n, w), 2: (n, u_count)}
    with torch.cuda.stream(stream):
        if write_volume and volume is None:
            volume = torch.empty((n, u_count, w), dtype=torch.uint16, device=dev)
        if not write_volume:
            volume = None
        if xy_u32 and (reduce != "max" or 0 not in axes or projections.get(0) is None):
            raise ParameterError("xy_u32 needs reduce='max' and a caller-owned projections[0] accumulator")
        for a in axes:
            t = projections.get(a)
            want = torch.int32 if (a == 0 and xy_u32) else pdt
            if t is None:
                t = (torch.zeros if (a == 0 and xy_accumulate) else torch.empty)(shapes[a], dtype=pdt, device=dev)
                projections[a] = t
            elif tuple(t.shape) != shapes[a] or t.dtype != want or not t.is_contiguous():
                raise ParameterError(f"projection {a} buffer must be contiguous {shapes[a]} {want}")
        if volume is not None and (tuple(volume.shape) != (n, u_count, w) or volume.dtype != torch.uint16):
            raise ParameterError(f"volume buffer must be (n, U, W) = {(n, u_count, w)} uint16")
        desc = make_desc(n, h, w, first_slice, shear_px, interp, formula, u_begin, u_count, reduce,
                         xy_accumulate, row_stride, frame_stride, xy_u32)
        lib = _lib.load()
        ws_bytes = int(lib.ssb_deskew_workspace_bytes(ctypes.byref(desc)))
        ws = _workspaces.get(ws_bytes, stream)
        _lib.check(lib.ssb_deskew(
            ctypes.byref(desc), _vp(raw), _vp(volume), _vp(projections.get(0)),
            _vp(projections.get(1)), _vp(projections.get(2)), _vp(ws), ctypes.c_size_t(ws.numel()),
            ctypes.c_void_p(stream.cuda_stream)))
    return DeskewResult(volume=volume, projections={a: projections[a] for a in axes},
                        canvas_rows=canvas_rows, u_begin=u_begin, u_count=u_count)


def deskew_batch(raw: torch.Tensor, shear_px: float, interp: str = "linear", *, formula: str = "canvas",
                 projection_axes=_AXES, reduce: str = "max", write_volume: bool = True,
                 volume: torch.Tensor | None = None, projections: dict | None = None,
                 stream: torch.cuda.Stream | None = None) -> DeskewResult:
    """Fused deskew + projections of B stacks of one shape in one launch (``ssb_deskew_batch``).

    raw: CUDA uint16 (B, n, H, W), C-contiguous.  Outputs carry a leading batch axis: volume
    (B, n, U, W); projections 0 -> (B, U, W), 1 -> (B, n, W), 2 -> (B, n, U).  Stack b's outputs
    equal ``deskew_device(raw[b], ...)``.  Small stacks (config 1) fill the GPU this way instead of
    one under-occupied launch per stack.
    """
    axes = check_options(interp, reduce, formula, projection_axes)
    if not isinstance(raw, torch.Tensor) or not raw.is_cuda or raw.dtype != torch.uint16 or raw.dim() != 4:
        raise ParameterError("raw must be a CUDA uint16 (B, n, H, W) tensor")
    if shear_px < 0:
        raise ParameterError(f"shear_px must be >= 0, got {shear_px}")
    raw = raw.contiguous()
    b, n, h, w = (int(v) for v in raw.shape)
    if b < 1 or n < 1:
        raise ParameterError("empty batch")
    u = canvas_rows_for(n, h, shear_px)
    dev = raw.device
    stream = stream or torch.cuda.current_stream(dev)
    pdt = proj_dtype(reduce)
    shapes = {0: (b, u, w), 1: (b, n, w), 2: (b, n, u)}
    projections = dict(projections or {})
    with torch.cuda.stream(stream):
        if write_volume and volume is None:
            volume = torch.empty((b, n, u, w), dtype=torch.uint16, device=dev)
        if not write_volume:
            volume = None
        for a in axes:
            t = projections.get(a)
            if t is None:
                projections[a] = torch.empty(shapes[a], dtype=pdt, device=dev)
            elif tuple(t.shape) != shapes[a] or t.dtype != pdt or not t.is_contiguous():
                raise ParameterError(f"projection {a} buffer must be contiguous {shapes[a]} {pdt}")
        if volume is not None and (tuple(volume.shape) != (b, n, u, w) or volume.dtype != torch.uint16
                                   or not volume.is_contiguous()):
            raise ParameterError(f"volume buffer must be contiguous (B, n, U, W) = {(b, n, u, w)} uint16")
        desc = make_desc(n, h, w, 0, shear_px, interp, formula, 0, u, reduce)
        lib = _lib.load()
        ws_bytes = int(lib.ssb_deskew_batch_workspace_bytes(ctypes.byref(desc), b))
        ws = _workspaces.get(ws_bytes, stream)
        _lib.check(lib.ssb_deskew_batch(
            ctypes.byref(desc), b, _vp(raw), _vp(volume), _vp(projections.get(0)), _vp(projections.get(1)),
            _vp(projections.get(2)), _vp(ws), ctypes.c_size_t(ws.numel()), ctypes.c_void_p(stream.cuda_stream)))
    return DeskewResult(volume=volume, projections={a: projections[a] for a in axes}, canvas_rows=u, u_begin=0,
                        u_count=u)


def frames_to_array(stack) -> np.ndarray:
    """Accept a list of RawFrame / 2-D arrays or an (n, H, W) array (ss/phantom.py:369-377)."""
    if isinstance(stack, np.ndarray) and stack.ndim == 3:
        if stack.dtype != np.uint16:
            raise ParameterError(f"frame pixels must be uint16, got {stack.dtype}")
        return stack
    frames = [f.pixels if hasattr(f, "pixels") else np.asarray(f) for f in stack]
    if not frames:
        raise ParameterError("empty stack")
    h, w = frames[0].shape
    for k, f in enumerate(frames):
        if f.shape != (h, w):
            raise ParameterError(f"frame {k} is {f.shape}, expected {(h, w)}")
    out = np.empty((len(frames), h, w), dtype=np.uint16)
    for k, f in enumerate(frames):
        out[k] = f
    return out


def deskew_volume(stack, geom, shear_px: float, interp: str = "linear", *,
                  projection_axes=_AXES, reduce: str = "max", write_volume: bool = True,
                  formula: str = "canvas", device_outputs: bool | None = None,
                  chunk_frames: int | None = None) -> DeskewResult:
    """Deskewed volume plus fused projections of one stack (north_star entry point).

    ``stack`` is a list of RawFrame / (H, W) uint16 arrays, an (n, H, W) uint16
    ndarray (pinned or pageable) or a torch uint16 tensor (CPU or CUDA).  Slice
    indices are the stack positions (ss/phantom.py:391); ``geom`` supplies the
    canvas-size limit (ss/geometry.py:129-147).  Host inputs stream through the
    pinned H2D pipeline; outputs come back to the host unless
    ``device_outputs`` is True (default: same side as the input).
    """
    from .geometry import DEFAULT_CANVAS_LIMIT_PX, output_extent
    from .stream import StackStreamer

    check_options(interp, reduce, formula, projection_axes)
    require_cuda()
    if isinstance(stack, torch.Tensor):
        if stack.dim() != 3:
            raise ParameterError("stack tensor must be (n, H, W)")
        if stack.dtype != torch.uint16:
            raise ParameterError(f"frame pixels must be uint16, got {stack.dtype}")
        n, h, w = (int(v) for v in stack.shape)
    else:
        stack = frames_to_array(stack)
        n, h, w = stack.shape
    if n == 0:
        raise ParameterError("empty stack")
    limit = DEFAULT_CANVAS_LIMIT_PX
    g = geom.with_frame(w, h) if geom is not None else None
    if g is not None:
        from dataclasses import replace
        output_extent(replace(g, slice_count=n), shear_px, limit)
    on_device = isinstance(stack, torch.Tensor) and stack.is_cuda
    if device_outputs is None:
        device_outputs = on_device
    if on_device:
        res = deskew_device(stack, shear_px, interp, formula=formula, projection_axes=projection_axes,
                            reduce=reduce, write_volume=write_volume)
    else:
        streamer = StackStreamer(h, w, chunk_frames=chunk_frames)
        res = streamer.run(stack, shear_px, interp, formula=formula, projection_axes=projection_axes,
                           reduce=reduce, write_volume=write_volume)
    if device_outputs:
        return res
    return DeskewResult(
        volume=None if res.volume is None else res.volume.cpu().numpy(),
        projections={a: t.cpu().numpy() for a, t in res.projections.items()},
        canvas_rows=res.canvas_rows, u_begin=res.u_begin, u_count=res.u_count)


class DeskewGraph:
    """One fixed-shape ``deskew_device`` call captured in a CUDA graph and replayed.

    For small stacks and fixed live-view geometries the scratch reset, the fused kernel and the
    finalize pass are replayed as one graph (config 1: 0.044 -> 0.041 ms per call,
    ``tools/graph_probe.py``).  The graph is bound to the buffers it was captured with: update
    ``raw`` in place between replays; ``replay()`` returns the same ``DeskewResult`` (its tensors
    are overwritten by every replay).
    """

    def __init__(self, raw: torch.Tensor, shear_px: float, interp: str = "linear", **kw):
        if "stream" in kw or "volume" in kw or "projections" in kw:
            raise ParameterError("DeskewGraph owns its stream and output buffers")
        self.raw = raw
        self.stream = torch.cuda.Stream(raw.device)
        self.stream.wait_stream(torch.cuda.current_stream(raw.device))
        self._args = (shear_px, interp)
        self._kw = kw
        # the first call allocates outputs and scratch; two more settle everything outside the graph
        self.result = deskew_device(raw, shear_px, interp, stream=self.stream, **kw)
        for _ in range(2):
            self._call()
        # the graph bakes in this stream's scratch buffer: hold it, so an LRU eviction from the
        # workspace cache cannot free memory the graph still writes
        self._workspace = _workspaces.get(1, self.stream)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._call()

    def _call(self):
        r = self.result
        kw = dict(self._kw)
        kw["write_volume"] = r.volume is not None
        deskew_device(self.raw, *self._args, volume=r.volume, projections=r.projections, stream=self.stream, **kw)

    def replay(self) -> DeskewResult:
        """Run the captured call on the caller's current stream order (waits for prior work)."""
        cur = torch.cuda.current_stream(self.raw.device)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            self.graph.replay()
        cur.wait_stream(self.stream)
        return self.result
