"""Rolling-mode refresh cost per camera frame on the GPU.

Times ProjectionCanvas.rolling_replace (ring of N frames in HBM, band re-max +
contributor map, ss/pipeline.py:345-377) per frame after a full sweep, and prints
one JSON line per configuration.  The reference measured 82.5 ms (nearest) and
270.6 ms (linear) per frame at config 1 on one CPU core.
"""

import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_00645_b200 import pipeline as pl  # noqa: E402
from paper_2211_00645_b200.geometry import SheetGeometry, native_shear_px  # noqa: E402
from paper_2211_00645_b200.stream import pinned_stack  # noqa: E402


def run(n, h, w, interp, frames=64):
    g = SheetGeometry(30.0, 0.115, 0.115, n, w, h)
    s = native_shear_px(g)
    c = pl.ProjectionCanvas(g, s, interp=interp, mode="rolling")
    rng = np.random.default_rng(0)
    pix = pinned_stack(n, h, w)  # camera frames land in page-locked buffers (ingest / StackStreamer)
    pix[:] = rng.integers(0, 4096, size=(n, h, w)).astype(np.uint16)
    for i in range(n):
        c.rolling_replace(pl.RawFrame(pix[i], i))
    c.stream.synchronize()
    # device time of the band kernel alone, and wall time per rolling_replace (incl. H2D)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(c.stream)
    for k in range(frames):
        i = (k * 37) % n
        c.rolling_replace(pl.RawFrame(pix[i], i, sweep_index=1))
    e1.record(c.stream)
    c.stream.synchronize()
    wall = (time.perf_counter() - t0) / frames * 1e3
    dev = e0.elapsed_time(e1) / frames
    # band update alone (ring already holds the frames): the two rolling kernels
    e0.record(c.stream)
    for k in range(frames):
        i = (k * 37) % n
        lo, hi = c.row_span(i)
        c._recompute_band(lo, hi, i)
    e1.record(c.stream)
    c.stream.synchronize()
    band = e0.elapsed_time(e1) / frames
    return {"config": f"{n}x{h}x{w}", "interp": interp, "ms_per_frame_wall": wall, "ms_per_frame_stream": dev,
            "ms_band_update": band}


if __name__ == "__main__":
    for (n, h, w) in ((128, 256, 512), (200, 1024, 1024), (512, 2048, 2048)):
        for interp in ("nearest", "linear"):
            print(json.dumps(run(n, h, w, interp, frames=64 if n < 512 else 16)), flush=True)
