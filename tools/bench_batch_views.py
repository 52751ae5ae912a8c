"""cli.run_batch's compute on the device: one warped MIP per view angle of a config-2 stack."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_00645_b200.batch import deskew_views  # noqa: E402
from paper_2211_00645_b200.geometry import SheetGeometry, view_transform  # noqa: E402
from paper_2211_00645_b200.stream import pinned_stack  # noqa: E402

n, h, w = 512, 2048, 2048
g = SheetGeometry(30.0, 0.115, 0.115, n, w, h)
host = pinned_stack(n, h, w)
host[:] = np.random.default_rng(0).integers(0, 4096, size=(n, h, w), dtype=np.uint16)
angles = (0.0, 15.0, 30.0, 45.0)
vts = [view_transform(g, view_angle_deg=a) for a in angles]
dev = torch.from_numpy(host).cuda()
for label, src in (("device-resident stack", dev), ("pinned host stack (H2D inside)", torch.from_numpy(host))):
    deskew_views(src, g, vts)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        imgs = deskew_views(src, g, vts)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    print(json.dumps({"what": "batch.deskew_views, 4 view angles, 512 x 2048 x 2048, images to host",
                      "input": label, "ms_per_stack": ms, "angles": angles,
                      "image_rows": [int(i.shape[0]) for i in imgs]}), flush=True)
