"""Display encode of the live view on the GPU: the frame packet of skewstream/server.py.

Drop-in for ``encode_frame_packet`` (ss/server.py:72-117).  The 64-byte header is packed on
the host (a handful of scalars); the payload comes from the device:

* ``gray16``: the little-endian uint16 image (server.py:93) -- a device image is copied down
  as is (B200 is little-endian, no conversion kernel);
* ``gray8``: ``ssb_encode_gray8`` -- min / max, ``rint((p - min) * (255 / range))`` and the
  byte pack in one cooperative launch (server.py:83-91); the header's ``g8_offset`` and
  ``g8_range`` come back with the bytes.

``image.pixels`` may be a numpy array (as the reference's DisplayImage holds) or a torch CUDA
tensor (the device canvas / warp output, no round trip through the host before encoding).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np
import torch

from . import _lib
from .deskew import require_cuda
from .errors import ParameterError

# wire format (ss/server.py:58-69)
MAGIC = b"SKWF"
VERSION = 1
HEADER_FMT = "<4sHBBHIIiIIIHHfffffIH"
HEADER_SIZE = struct.calcsize(HEADER_FMT)
PIXEL_FORMATS = {"gray16": 0, "gray8": 1}
MODES = {"global": 0, "rolling": 1}
_MAX_DIM = 2**31 - 1

def _stats_buffer(device: torch.device) -> torch.Tensor:
    """A fresh result buffer per call (caching allocator, on the current stream): a later encode on
    the same stream cannot overwrite the (g8_offset, g8_range) a caller has not read yet."""
    nbytes = int(_lib.load().ssb_encode_gray8_stats_bytes())
    return torch.empty(nbytes // 4, dtype=torch.int32, device=device)


def _as_device_u16(pixels) -> torch.Tensor:
    if isinstance(pixels, torch.Tensor):
        if not pixels.is_cuda:
            pixels = pixels.to(require_cuda())
        t = pixels
    else:
        a = np.ascontiguousarray(np.asarray(pixels), dtype=np.uint16)
        t = torch.from_numpy(a.view(np.int16)).to(require_cuda()).view(torch.uint16)
    if t.dtype not in (torch.uint16, torch.int16):
        raise ParameterError(f"display pixels must be uint16, got {t.dtype}")
    return t.contiguous()


def encode_gray8_device(pixels, stream: torch.cuda.Stream | None = None):
    """gray8 payload of a uint16 image on the device.

    Returns ``(payload, stats)``: ``payload`` uint8 with the image's shape, ``stats`` a device
    int32 tensor whose first two words are the header's (g8_offset, g8_range).  Asynchronous on
    ``stream`` (default: the current stream).  An empty image raises ValueError, as numpy's
    ``min()`` does in the reference.
    """
    dev = pixels.device if isinstance(pixels, torch.Tensor) and pixels.is_cuda else require_cuda()
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    producer = torch.cuda.current_stream(dev)
    if st != producer:
        st.wait_stream(producer)  # a device image written on the caller's stream is complete
    with torch.cuda.stream(st):  # upload / contiguous copy ordered before the kernel on `st`
        t = _as_device_u16(pixels)
    if t.numel() == 0:
        raise ValueError("zero-size array to reduction operation minimum which has no identity")
    if st != producer and isinstance(pixels, torch.Tensor) and pixels.is_cuda:
        t.record_stream(st)  # the caller's tensor may be freed while `st` still reads it
    lib = _lib.load()
    with torch.cuda.stream(st):
        stats = _stats_buffer(t.device)
        out = torch.empty(t.shape, dtype=torch.uint8, device=t.device)
    _lib.check(lib.ssb_encode_gray8(ctypes.c_void_p(t.data_ptr()), t.numel(), ctypes.c_void_p(out.data_ptr()),
                                    ctypes.c_void_p(stats.data_ptr()), stats.numel() * 4,
                                    ctypes.c_void_p(st.cuda_stream)))
    return out, stats


def frame_header(image, pixel_format: str, g8_offset: int = 0, g8_range: int = 0,
                 telemetry: dict | None = None) -> bytes:
    """The 64-byte packet header (field order of ss/server.py:94-115)."""
    h, w = (int(v) for v in image.pixels.shape)
    t = image.timings
    tele = telemetry or {}
    return struct.pack(
        HEADER_FMT, MAGIC, VERSION, PIXEL_FORMATS[pixel_format], MODES.get(image.mode, 0),
        image.channel_id, image.sweep_index, image.slice_index,
        int(round(image.view_angle_deg * 100)), w, h, int(round(image.out_pitch_um * 1000)),
        g8_offset, g8_range,
        t.acquisition_ms if t else 0.0, t.processing_ms if t else 0.0,
        t.plotting_ms if t else 0.0, t.lag_ms if t else 0.0,
        float(tele.get("fps", 0.0)),
        int(sum(tele.get("drops", {}).values())) if "drops" in tele else 0,
        0,
    )


def encode_frame_packet(image, pixel_format: str = "gray16", telemetry: dict | None = None) -> bytes:
    """Serialize one display frame (ss/server.py:72-117), payload encoded on the GPU."""
    if pixel_format not in PIXEL_FORMATS:
        raise ParameterError(f"unknown pixel format {pixel_format!r}")
    h, w = (int(v) for v in image.pixels.shape)
    if w > _MAX_DIM or h > _MAX_DIM:
        raise ParameterError(f"image {w}x{h} exceeds header field range")
    if pixel_format == "gray8":
        payload, stats = encode_gray8_device(image.pixels)
        host = torch.empty(payload.numel() + 8, dtype=torch.uint8, pin_memory=True)
        host[:payload.numel()].copy_(payload.view(-1), non_blocking=True)
        host[payload.numel():].copy_(stats[:2].view(torch.uint8), non_blocking=True)
        torch.cuda.current_stream(payload.device).synchronize()
        off, rng = np.frombuffer(host[payload.numel():].numpy().tobytes(), dtype="<u4")
        return frame_header(image, pixel_format, int(off), int(rng), telemetry) + host[:payload.numel()].numpy().tobytes()
    px = image.pixels
    if isinstance(px, torch.Tensor):
        body = px.contiguous().view(torch.int16).cpu().numpy().tobytes()
    else:
        body = np.asarray(px).astype("<u2").tobytes()
    return frame_header(image, pixel_format, 0, 0, telemetry) + body
