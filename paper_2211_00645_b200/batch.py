"""Multi-view batch projections: the compute of skewstream's ``cli.run_batch`` on the device.

``run_batch`` (ss/cli.py:308-338) deskews a recorded stack into one max projection per requested
view angle: for every ``ViewTransform`` it builds a ``ProjectionCanvas`` at that shear, places all
N frames, finalizes, and warps the canvas (``warp_projection``, ss/pipeline.py:434-457) -- N
placements per angle.  Here the stack crosses PCIe once (pinned, chunked when it comes from the
host), and each view is one fused XY-only launch at its shear plus one device warp, on one stream.
File writing, PNG encoding and the metadata manifest stay with the caller (control plane).

The result of each view is bit-identical to the reference's ``warp_projection(
ProjectionCanvas(...).finalize_global(), vt.warp_scale)`` (tests/test_gpu_acceptance.py checks
it against the reference's own images for four view angles).
"""

from __future__ import annotations

import threading
from dataclasses import replace

import numpy as np
import torch

from .deskew import deskew_device, frames_to_array, require_cuda
from .errors import ParameterError
from .geometry import SheetGeometry, ViewTransform, output_extent
from .pipeline import warp_projection_device


def deskew_views(stack, geom: SheetGeometry, transforms, interp: str = "linear", *,
                 device_outputs: bool = False) -> list:
    """One warped max projection per view transform (the images ``cli.run_batch`` writes).

    ``stack``: list of RawFrame / (H, W) arrays, an (n, H, W) uint16 array, or a torch uint16
    tensor (host or CUDA).  ``transforms``: ``ViewTransform``s (``geometry.view_transform``).
    Returns uint16 (rows, W) images, host numpy arrays unless ``device_outputs``.
    """
    dev = require_cuda()
    if isinstance(stack, torch.Tensor):
        if stack.dtype != torch.uint16 or stack.dim() != 3:
            raise ParameterError("stack tensor must be (n, H, W) uint16")
        raw = stack if stack.is_cuda else stack.to(dev, non_blocking=stack.is_pinned())
    else:
        raw = torch.from_numpy(frames_to_array(stack)).to(dev)
    n, h, w = (int(v) for v in raw.shape)
    if n == 0:
        raise ParameterError("empty stack")
    g = replace(geom.with_frame(w, h), slice_count=n)
    transforms = list(transforms)
    if not all(isinstance(vt, ViewTransform) for vt in transforms):
        raise ParameterError("transforms must be ViewTransform objects")
    stream = torch.cuda.current_stream(dev)
    images = []
    for vt in transforms:
        _, rows = output_extent(g, vt.shear_px)  # the reference's canvas size and limit check
        res = deskew_device(raw, vt.shear_px, interp, canvas_rows=rows, projection_axes=(0,),
                            write_volume=False, stream=stream)
        images.append(warp_projection_device(res.projections[0], vt.warp_scale, stream))
    if device_outputs:
        return images
    # one reused page-locked landing buffer (a fresh pinned allocation per call costs more than the
    # copies); all images land in it with async copies, then one synchronisation and host copies out
    sizes = [t.numel() for t in images]
    with _STAGING_LOCK:
        buf = _STAGING.get(dev.index)
        if buf is None or buf.numel() < sum(sizes):
            buf = _STAGING[dev.index] = torch.empty(sum(sizes), dtype=torch.int16, pin_memory=True)
        off = 0
        for t, k in zip(images, sizes):
            buf[off:off + k].copy_(t.reshape(-1).view(torch.int16), non_blocking=True)
            off += k
        stream.synchronize()
        out, off = [], 0
        for t, k in zip(images, sizes):
            out.append(buf[off:off + k].numpy().view(np.uint16).reshape(tuple(t.shape)).copy())
            off += k
    return out


_STAGING: dict = {}
_STAGING_LOCK = threading.Lock()
