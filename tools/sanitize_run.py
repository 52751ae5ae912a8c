"""Small end-to-end exercise of every libssb kernel for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_00645_b200 import pipeline as pl  # noqa: E402
from paper_2211_00645_b200.deskew import deskew_device  # noqa: E402
from paper_2211_00645_b200.geometry import SheetGeometry  # noqa: E402

rng = np.random.default_rng(0)
for (n, h, w, s) in ((24, 40, 264, 0.866), (7, 9, 17, 0.5), (33, 130, 512, 0.7071)):
    st = torch.from_numpy(rng.integers(0, 65536, (n, h, w)).astype(np.uint16)).cuda()
    for interp in ("linear", "nearest"):
        for formula in ("canvas", "npinterp"):
            for reduce in ("max", "sum"):
                for vol in (True, False):
                    deskew_device(st, s, interp, formula=formula, reduce=reduce, write_volume=vol)
torch.cuda.synchronize()
g = SheetGeometry(60.0, 0.2, 0.1, 6, 24, 10)
c = pl.ProjectionCanvas(g, 1.3, interp="linear", mode="rolling")
for k in range(12):
    c.rolling_replace(pl.RawFrame(rng.integers(0, 4, (10, 24)).astype(np.uint16), k % 6))
c.replace_all(0.9)
pl.warp_projection(c.max_pixels, 1.37)
torch.cuda.synchronize()
print("sanitize run ok")
