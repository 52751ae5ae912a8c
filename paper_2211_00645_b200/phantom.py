"""Drop-in for ``skewstream.phantom.reference_deskew`` (ss/phantom.py:359-402) on B200.

The reference materialises an (n, U, W) float64 pile with np.interp per column
and reduces it with one max; here one fused kernel computes the same rounded
values (np.interp restated in fp64, bit-exact) and the XY max without ever
materialising the pile.  The rest of ``skewstream.phantom`` (scene rendering,
rotation oracle, PNG IO) is test-data generation and stays out of scope.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import torch

from . import geometry
from .deskew import deskew_device, frames_to_array, require_cuda
from .errors import ParameterError
from .geometry import SheetGeometry

MAX_INTENSITY = 65535  # ss/phantom.py:34


def reference_deskew(stack, geom: SheetGeometry, shear_px: float, interp: str = "nearest") -> np.ndarray:
    """Whole-stack deskew -> XY max projection, uint16 (ss/phantom.py:359-402).

    Slice offsets use the position in ``stack`` (ss/phantom.py:391); when the
    stack length differs from ``geom.slice_count`` the canvas is re-derived
    from the stack (ss/phantom.py:378-389).
    """
    if interp not in ("nearest", "linear"):
        raise ParameterError(f"interp must be nearest or linear, got {interp!r}")
    if isinstance(stack, torch.Tensor) and stack.is_cuda:
        raw = stack
        n, h, w = (int(v) for v in raw.shape)
        if n == 0:
            raise ParameterError("empty stack")
    else:
        arr = frames_to_array(stack)
        n, h, w = arr.shape
        if n == 0:
            raise ParameterError("empty stack")
        raw = torch.from_numpy(np.ascontiguousarray(arr)).to(require_cuda())
    canvas_geom = replace(geom.with_frame(w, h), slice_count=n)
    width, height = geometry.output_extent(canvas_geom, shear_px)
    res = deskew_device(raw, shear_px, interp, formula="npinterp", canvas_rows=height,
                        projection_axes=(0,), write_volume=False)
    xy = res.projections[0]
    if isinstance(stack, torch.Tensor) and stack.is_cuda:
        return xy
    return xy.cpu().numpy()
