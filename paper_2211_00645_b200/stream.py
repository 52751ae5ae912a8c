"""Pinned-memory, multi-stream host-to-device pipeline (north_star subsystem 3).

Replaces the reference's acquisition -> per-channel deskew worker hand-off
(``LivePipeline._acquire_loop`` / ``_deskew_loop``, ss/pipeline.py:1020-1055,
and the paper's multiprocessing workers) for continuous acquisition: frames are
cut into chunks, each chunk is copied host -> device on one of two copy
streams while the previous chunk is being deskewed on the compute stream, and
the projections accumulate on device (XY folds chunk after chunk with
``SSB_FLAG_XY_ACCUMULATE``; XZ / YZ rows of a chunk are written in place).

* Pinned inputs (``pinned_stack()``, or any page-locked torch CPU tensor) are
  copied straight from the caller's buffer.
* Pageable inputs are first staged into a ring of pinned buffers (one host
  memcpy per chunk) -- that is what a camera driver's DMA ring replaces.
"""

from __future__ import annotations

import os
import time
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np
import torch

from .deskew import DeskewResult, canvas_rows_for, check_options, deskew_device, proj_dtype, require_cuda
from .errors import ParameterError


def _parse_cpulist(text: str) -> set:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus


def gpu_numa_cpus(device=None):
    """Host CPUs of the GPU's NUMA node (sysfs, intersected with this thread's affinity), or
    None when the platform does not say (single-node hosts, containers without sysfs)."""
    try:
        p = torch.cuda.get_device_properties(torch.device("cuda", torch.cuda.current_device())
                                             if device is None else device)
        pci = "/sys/bus/pci/devices/%04x:%02x:%02x.0/numa_node" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        with open(pci) as f:
            node = int(f.read())
        if node < 0:
            return None
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            cpus = _parse_cpulist(f.read()) & os.sched_getaffinity(0)
        return cpus or None
    except (OSError, ValueError, AttributeError, RuntimeError, AssertionError):
        return None


@contextmanager
def near_gpu(device=None):
    """Run the body on the GPU's NUMA node (this thread only, restored afterwards).

    Page-locked buffers allocated inside land in that node's memory (local first-touch
    policy), so the copy engines read them without crossing the socket link: on a
    two-socket host a remote pinned stack copies at ~33 GB/s instead of ~55 GB/s."""
    cpus = gpu_numa_cpus(device)
    if cpus is None:
        yield
        return
    old = os.sched_getaffinity(0)
    os.sched_setaffinity(0, cpus)
    try:
        yield
    finally:
        os.sched_setaffinity(0, old)


def pinned_stack(n: int, height: int, width: int, device=None) -> np.ndarray:
    """(n, H, W) uint16 numpy array backed by page-locked host memory on ``device``'s NUMA node."""
    require_cuda()
    with near_gpu(device):
        t = torch.empty((n, height, width), dtype=torch.uint16, pin_memory=True)
    return t.numpy()  # the array's base holds the tensor: the pinned block lives as long as the array


def _as_host_tensor(stack) -> torch.Tensor:
    if isinstance(stack, torch.Tensor):
        if stack.is_cuda:
            raise ParameterError("StackStreamer takes host frames; use deskew_device for CUDA tensors")
        return stack
    arr = np.ascontiguousarray(stack)
    if arr.dtype != np.uint16 or arr.ndim != 3:
        raise ParameterError("stack must be an (n, H, W) uint16 array")
    return torch.from_numpy(arr)


def chunk_bounds(n: int, chunk: int, tail: int) -> list:
    """[c0, c1) frame ranges: full chunks, the last one split so it holds <= ``tail`` frames."""
    bounds = [(c0, min(n, c0 + chunk)) for c0 in range(0, n, chunk)]
    if bounds and bounds[-1][1] - bounds[-1][0] > tail:
        c0, c1 = bounds.pop()
        bounds += [(c0, c1 - tail), (c1 - tail, c1)]
    return bounds


@dataclass
class StreamTimings:
    """Host-side wall times of the last run (ms)."""

    total_ms: float = 0.0
    last_chunk_ready_to_done_ms: float = 0.0


class StackStreamer:
    """Chunked H2D + deskew pipeline for one frame geometry (H, W)."""

    def __init__(self, height: int, width: int, *, chunk_frames: int | None = None,
                 tail_frames: int | None = None, n_buffers: int = 3, device: torch.device | None = None):
        self.device = device or require_cuda()
        self.height, self.width = int(height), int(width)
        frame_bytes = 2 * self.height * self.width
        if chunk_frames is None:
            # 64 MB chunks: measured on B200 (config 3, 200 x 1024^2): 16-64 MB chunks keep the
            # PCIe link saturated (7.65 ms/stack), 128-256 MB chunks stall it (11-13.6 ms)
            chunk_frames = max(1, (64 << 20) // frame_bytes)
        if tail_frames is None:
            # the last chunk is cut to <= 16 MB: it is the one whose copy + deskew + D2H is the
            # live view's latency (last frame on the host -> projections on the host)
            tail_frames = max(1, (16 << 20) // frame_bytes)
        self.chunk = int(chunk_frames)
        self.tail = max(1, min(int(tail_frames), self.chunk))
        self.n_buffers = max(2, int(n_buffers))
        shape = (self.chunk, self.height, self.width)
        self.dev_bufs = [torch.empty(shape, dtype=torch.uint16, device=self.device)
                         for _ in range(self.n_buffers)]
        self._staging = None  # pinned ring, allocated on first pageable input
        self.copy_streams = [torch.cuda.Stream(self.device) for _ in range(2)]
        self.compute_stream = torch.cuda.Stream(self.device)
        self._done = [None] * self.n_buffers  # compute-finished events per buffer
        self.timings = StreamTimings()
        #: if set to a timing-enabled torch.cuda.Event, run() records it on the copy stream
        #: right before the last chunk's H2D copy (end-to-end latency measurement)
        self.last_chunk_event = None

    def chunk_bounds(self, n: int) -> list:
        return chunk_bounds(n, self.chunk, self.tail)

    def _staging_ring(self):
        if self._staging is None:
            shape = (self.chunk, self.height, self.width)
            with near_gpu(self.device):
                self._staging = [torch.empty(shape, dtype=torch.uint16, pin_memory=True)
                                 for _ in range(self.n_buffers)]
        return self._staging

    def run(self, stack, shear_px: float, interp: str = "linear", *, formula: str = "canvas",
            projection_axes=(0, 1, 2), reduce: str = "max", write_volume: bool = True,
            first_slice: int = 0, canvas_rows: int | None = None, out: DeskewResult | None = None
            ) -> DeskewResult:
        """Deskew a host stack chunk by chunk; returns device outputs (not synchronised
        with the host; the caller's current stream is made to wait for them)."""
        axes = check_options(interp, reduce, formula, projection_axes)
        src = _as_host_tensor(stack)
        n, h, w = (int(v) for v in src.shape)
        if (h, w) != (self.height, self.width):
            raise ParameterError(f"frames are {(h, w)}, streamer built for {(self.height, self.width)}")
        if n == 0:
            raise ParameterError("empty stack")
        if canvas_rows is None:
            canvas_rows = canvas_rows_for(first_slice + n, h, shear_px)
        pinned = src.is_pinned()
        dev = self.device
        t0 = time.perf_counter()
        pdt = proj_dtype(reduce)
        with torch.cuda.stream(self.compute_stream):
            if out is None:
                volume = torch.empty((n, canvas_rows, w), dtype=torch.uint16, device=dev) if write_volume else None
                shapes = {0: (canvas_rows, w), 1: (n, w), 2: (n, canvas_rows)}
                projs = {a: torch.empty(shapes[a], dtype=pdt, device=dev) for a in axes}
            else:
                volume, projs = out.volume, dict(out.projections)
        bounds = self.chunk_bounds(n)
        n_chunks = len(bounds)
        # max-mode XY: one int32 accumulator for the whole stack (SSB_FLAG_XY_U32), narrowed once
        # at the end, instead of a whole-canvas scratch reset + narrowing pass per chunk
        acc32 = None
        if reduce == "max" and 0 in axes and n_chunks > 1 and w % 8 == 0:
            with torch.cuda.stream(self.compute_stream):
                acc32 = torch.zeros((canvas_rows, w), dtype=torch.int32, device=dev)
        for c, (c0, c1) in enumerate(bounds):
            b = c % self.n_buffers
            m = c1 - c0
            cs = self.copy_streams[c % 2]
            if self._done[b] is not None:
                if not pinned:
                    # the staging slot is free once the deskew that consumed it finished
                    self._done[b].synchronize()
                cs.wait_event(self._done[b])
            if pinned:
                host = src[c0:c1]
            else:
                host = self._staging_ring()[b][:m]
                host.copy_(src[c0:c1])  # pageable -> pinned (host memcpy)
            with torch.cuda.stream(cs):
                if c == n_chunks - 1 and self.last_chunk_event is not None:
                    self.last_chunk_event.record(cs)
                self.dev_bufs[b][:m].copy_(host, non_blocking=True)
                copied = torch.cuda.Event()
                copied.record(cs)
            self.compute_stream.wait_event(copied)
            chunk_projs = {}
            if 0 in axes:
                chunk_projs[0] = projs[0] if acc32 is None else acc32
            if 1 in axes:
                chunk_projs[1] = projs[1][c0:c1]
            if 2 in axes:
                chunk_projs[2] = projs[2][c0:c1]
            deskew_device(self.dev_bufs[b][:m], shear_px, interp, formula=formula,
                          first_slice=first_slice + c0, canvas_rows=canvas_rows,
                          projection_axes=axes, reduce=reduce, write_volume=write_volume,
                          volume=None if volume is None else volume[c0:c1],
                          projections=chunk_projs, xy_accumulate=c > 0 and acc32 is None,
                          xy_u32=acc32 is not None, stream=self.compute_stream)
            done = torch.cuda.Event()
            done.record(self.compute_stream)
            self._done[b] = done
        if acc32 is not None:
            with torch.cuda.stream(self.compute_stream):
                projs[0].copy_(acc32)  # values <= 65535: exact narrowing
        current = torch.cuda.current_stream(dev)
        current.wait_stream(self.compute_stream)
        for t in [volume, *projs.values()]:
            if t is not None:
                t.record_stream(current)
        self.timings.total_ms = (time.perf_counter() - t0) * 1e3
        return DeskewResult(volume=volume, projections=projs, canvas_rows=canvas_rows,
                            u_begin=0, u_count=canvas_rows)
