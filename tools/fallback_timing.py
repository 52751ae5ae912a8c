"""Time the generic tiled fallback against the TMA kernel on config-2-sized stacks."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00645_b200.deskew import deskew_device  # noqa: E402

s = math.cos(math.radians(30.0))
for w, disable in ((2048, "0"), (2048, "1"), (2044, "0"), (2046, "0"), (2047, "0")):
    os.environ["SSB_DISABLE_TMA"] = disable
    raw = torch.randint(0, 4096, (512, 2048, w), dtype=torch.int32, device="cuda").to(torch.uint16)
    res = deskew_device(raw, s, "linear")
    for _ in range(2):
        deskew_device(raw, s, "linear", volume=res.volume, projections=res.projections)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        deskew_device(raw, s, "linear", volume=res.volume, projections=res.projections)
    e1.record()
    torch.cuda.synchronize()
    print(f"W={w} SSB_DISABLE_TMA={disable}: {e0.elapsed_time(e1) / 5:.3f} ms/call")
    del raw, res
