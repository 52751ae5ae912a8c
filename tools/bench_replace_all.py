"""Rolling-mode replace_all (view change) cost on the GPU, config 1 / 3 / 2 sizes."""
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
    c = pl.ProjectionCanvas(g, s, interp="linear", mode="rolling")
    pix = pinned_stack(n, h, w)
    pix[:] = np.random.default_rng(0).integers(0, 4096, size=(n, h, w)).astype(np.uint16)
    for i in range(n):
        c.rolling_replace(pl.RawFrame(pix[i], i))
    c.stream.synchronize()
    t0 = time.perf_counter()
    c.replace_all(s * 0.9)
    c.stream.synchronize()
    t1 = time.perf_counter()
    print(json.dumps({"config": f"{n}x{h}x{w}", "replace_all_ms": (t1 - t0) * 1e3}), flush=True)
