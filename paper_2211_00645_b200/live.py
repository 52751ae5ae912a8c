"""Device side of one live-view channel: the deskew stage of skewstream's LivePipeline on B200.

The reference's threaded pipeline (ss/pipeline.py:706-1064) hands each channel's frames to
``_process_channel_frame`` (:900-947) and the result to ``_finish_emission`` (:951-980), both
driving a ``ProjectionCanvas``.  Its threads, queues, mailboxes and telemetry are control
plane and stay out of scope; this module is the per-channel GPU work between them:

* one device ``ProjectionCanvas`` per channel, on that canvas's own CUDA stream;
* the reference's sweep bookkeeping: global mode accumulates a sweep and emits when all N
  slices are placed (a new sweep index abandons a partial sweep; a pending view transform is
  applied at the sweep boundary through ``replace_all``); rolling mode refreshes the band of
  every frame and emits each time;
* ``StageTimings`` from CUDA events on the canvas stream: ``processing_ms`` is the device time
  of the sweep's placement launches (global) or of the last N band refreshes (rolling),
  ``plotting_ms`` the warp, ``acquisition_ms`` the stack period from frame timestamps and
  ``lag_ms`` host time from the last slice's timestamp to emission (ss/pipeline.py:973).

``process`` returns a ``DisplayImage`` (pixels on the host as in the reference, or left on the
device with ``device_pixels=True`` for ``display.encode_frame_packet``) or None.
"""

from __future__ import annotations

import time
from collections import deque

import numpy as np
import torch

from .errors import ParameterError
from .geometry import SheetGeometry, ViewTransform
from .pipeline import DisplayImage, ProjectionCanvas, RawFrame, StageTimings, warp_projection_device


class ChannelDeskewer:
    """One channel's canvas + stream + timings (ss/pipeline.py:680-700 ``_ChannelState``)."""

    def __init__(self, channel_id: int, geom: SheetGeometry, vt: ViewTransform, interp: str = "linear",
                 mode: str = "global", *, clock_ns=time.monotonic_ns, device_pixels: bool = False):
        self.channel_id = channel_id
        self.geom = geom
        self.vt = vt
        self.pending_vt: ViewTransform | None = None
        self.mode = mode
        self.canvas = ProjectionCanvas(geom, vt.shear_px, interp, mode)
        self.stream = self.canvas.stream
        self.clock_ns = clock_ns
        self.device_pixels = device_pixels
        self.current_sweep = -1
        self.waiting_for_sweep_start = False
        n = geom.slice_count
        self.frame_ts: deque = deque(maxlen=n + 1)
        self._sweep_events: list = []        # (start, end) per placement of the current sweep
        self._frame_proc_ms: deque = deque(maxlen=n)  # rolling: device ms of the last N refreshes
        self._frame_plot_ms: deque = deque(maxlen=n)

    # -- parameters (ss/pipeline.py:850-871, applied at a frame boundary) -------------------
    def set_mode(self, mode: str) -> None:
        if mode not in ("global", "rolling"):
            raise ParameterError(f"mode must be global or rolling, got {mode!r}")
        if mode == self.mode:
            return
        self.mode = mode
        self.canvas.mode = mode
        self.canvas.reset()
        self.canvas.ring = [None] * self.geom.slice_count
        self.waiting_for_sweep_start = mode == "global"
        self.current_sweep = -1

    def set_view(self, vt: ViewTransform) -> None:
        if self.mode == "rolling":
            self.vt = vt
            self.canvas.replace_all(vt.shear_px)
        else:
            self.pending_vt = vt

    def stack_period_ms(self) -> float:
        ts = self.frame_ts
        if len(ts) < 2:
            return 0.0
        return (ts[-1] - ts[0]) / 1e6 * (self.geom.slice_count / (len(ts) - 1))

    # -- per-frame work -----------------------------------------------------------------
    def _timed(self, fn):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        out = fn()
        e1.record(self.stream)
        return out, (e0, e1)

    def process(self, frame: RawFrame) -> DisplayImage | None:
        """``_process_channel_frame`` + ``_finish_emission`` for one frame of this channel."""
        n = self.geom.slice_count
        self.frame_ts.append(frame.timestamp_ns)
        if self.mode == "global":
            if self.waiting_for_sweep_start:
                if frame.slice_index != 0:
                    return None
                self.waiting_for_sweep_start = False
            if frame.sweep_index != self.current_sweep:
                if self.pending_vt is not None:
                    self.vt, self.pending_vt = self.pending_vt, None
                    self.canvas.replace_all(self.vt.shear_px)
                else:
                    self.canvas.reset()
                self.current_sweep = frame.sweep_index
                self._sweep_events = []
            _, ev = self._timed(lambda: self.canvas.place(frame))
            self._sweep_events.append(ev)
            if self.canvas.placed_count < n:
                return None
            projection, ev = self._timed(self.canvas.finalize_global_device)
            self._sweep_events.append(ev)
            proc_events = self._sweep_events
        else:
            if frame.sweep_index != self.current_sweep:
                self.current_sweep = frame.sweep_index
            _, ev = self._timed(lambda: self.canvas.rolling_replace(frame))
            with torch.cuda.stream(self.stream):
                projection = self.canvas.max_pixels_device.clone()
            proc_events = [ev]
        image, pev = self._timed(lambda: warp_projection_device(projection, self.vt.warp_scale, self.stream))
        pev[1].synchronize()
        # each event pair is read once (an elapsed_time call per pair); rolling mode keeps the
        # last N refreshes as numbers, as the reference keeps its per-exposure durations
        processing_ms = sum(a.elapsed_time(b) for a, b in proc_events)
        if self.mode == "rolling":
            self._frame_proc_ms.append(processing_ms)
            processing_ms = sum(self._frame_proc_ms)
            self._frame_plot_ms.append(pev[0].elapsed_time(pev[1]))
            plotting_ms = sum(self._frame_plot_ms)
        else:
            plotting_ms = pev[0].elapsed_time(pev[1])
        if self.device_pixels:
            pixels = image
        else:
            # page-locked landing buffer (cached by torch's host allocator), owned by the image
            host = torch.empty(tuple(image.shape), dtype=torch.int16, pin_memory=True)
            with torch.cuda.stream(self.stream):  # the copy and the event on the canvas stream
                host.copy_(image.view(torch.int16), non_blocking=True)
                host_done = torch.cuda.Event()
                host_done.record(self.stream)
            host_done.synchronize()
            pixels = host.numpy().view(np.uint16)
        t1 = self.clock_ns()
        timings = StageTimings(acquisition_ms=self.stack_period_ms(), processing_ms=processing_ms,
                               plotting_ms=plotting_ms, lag_ms=max(0.0, (t1 - frame.timestamp_ns) / 1e6))
        return DisplayImage(pixels=pixels, channel_id=frame.channel_id, sweep_index=frame.sweep_index,
                            slice_index=frame.slice_index, view_angle_deg=self.vt.view_angle_deg,
                            mode=self.mode, out_pitch_um=self.vt.out_pitch_um,
                            lateral_pitch_um=self.geom.pixel_pitch_um, timings=timings, emitted_at_ns=t1)
