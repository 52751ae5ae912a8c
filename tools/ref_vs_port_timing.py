"""Calibrate the bench's CPU arm: the reference's own ProjectionCanvas.place (run here, where
/root/reference is importable) against the oracle port bench.py times on the GPU box, on the
same frames of config 2, single process.  Writes profiles/r01_ref_vs_port_timing.json.

    PYTHONPATH=/root/reference/pkg/src python tools/ref_vs_port_timing.py
"""
import json
import math
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import deskew_oracle as O  # noqa: E402
from skewstream import geometry as G  # noqa: E402  (the reference)
from skewstream import pipeline as PL  # noqa: E402

n, h, w, frames = 512, 2048, 2048, 6
g = G.SheetGeometry(alpha_deg=30.0, scan_step_um=0.115, pixel_pitch_um=0.115, slice_count=n,
                    frame_width_px=w, frame_height_px=h)
s = G.native_shear_px(g)
rng = np.random.default_rng(0)
stack = rng.integers(0, 4096, size=(frames, h, w)).astype(np.uint16)
first = n // 2
out = {"config": "config2 frames 2048x2048, linear, slices %d..%d" % (first, first + frames - 1)}
for interp in ("linear", "nearest"):
    c = PL.ProjectionCanvas(g, s, interp=interp)
    t0 = time.perf_counter()
    for k in range(frames):
        c.place(PL.RawFrame(stack[k], first + k))
    t_ref = (time.perf_counter() - t0) / frames
    canvas = np.zeros((c.height, w), dtype=np.uint16)
    t0 = time.perf_counter()
    for k in range(frames):
        lo, hi, rows = O.slice_rows(stack[k], first + k, s, interp, "canvas")
        np.maximum(canvas[lo:hi + 1], rows, out=canvas[lo:hi + 1])
    t_port = (time.perf_counter() - t0) / frames
    same = bool(np.array_equal(canvas, c.max_pixels))
    out[interp] = {"reference_ms_per_frame": t_ref * 1e3, "port_ms_per_frame": t_port * 1e3,
                   "port_over_reference_speed": t_ref / t_port, "same_canvas": same}
    print(interp, out[interp], flush=True)
json.dump(out, open(os.path.join(REPO, "profiles", "r01_ref_vs_port_timing.json"), "w"), indent=1)
