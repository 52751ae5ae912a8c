"""Per-frame cost of the drop-in ProjectionCanvas.place (the LivePipeline path, ss/pipeline.py:918)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_00645_b200 import pipeline as pl  # noqa: E402
from paper_2211_00645_b200.geometry import SheetGeometry, native_shear_px  # noqa: E402
from paper_2211_00645_b200.stream import pinned_stack  # noqa: E402

for (n, h, w) in ((128, 256, 512), (200, 1024, 1024), (512, 2048, 2048)):
    g = SheetGeometry(30.0, 0.115, 0.115, n, w, h)
    s = native_shear_px(g)
    host = pinned_stack(n, h, w)
    host[:] = np.random.default_rng(0).integers(0, 4096, size=(n, h, w), dtype=np.uint16)
    pageable = np.array(host)
    for label, src in (("pinned", host), ("pageable", pageable)):
        c = pl.ProjectionCanvas(g, s, interp="linear")
        for i in range(n):  # warm-up sweep
            c.place(pl.RawFrame(src[i], i))
        c.finalize_global()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n):
            c.place(pl.RawFrame(src[i], i))
        out = c.finalize_global()
        dt = (time.perf_counter() - t0) / n * 1e3
        print(json.dumps({"config": f"{n}x{h}x{w}", "frames": label, "ms_per_place": dt,
                          "stack_ms": dt * n}), flush=True)
