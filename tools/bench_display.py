"""Time the display encode (gray8, one cooperative launch) on a config-2 canvas (2491 x 2048)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00645_b200 import display as D  # noqa: E402

for rows, cols in ((2491, 2048), (1197, 1024)):
    img = torch.randint(0, 65536, (rows, cols), dtype=torch.int32, device="cuda").to(torch.uint16)
    for _ in range(5):
        D.encode_gray8_device(img)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 200
    e0.record()
    for _ in range(iters):
        D.encode_gray8_device(img)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    nbytes = img.numel() * 3  # u16 read once from HBM + u8 written (2nd read hits L2)
    print(f"gray8 encode {rows}x{cols}: {us:.1f} us/call (incl. launch), {nbytes / us / 1e3:.0f} GB/s algorithmic")
