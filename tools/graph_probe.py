"""Config-1-sized fused deskew: direct launches vs CUDA-graph replay (L2 flushed before each step)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00645_b200.deskew import deskew_device  # noqa: E402

n, h, w = 128, 256, 512
s = math.cos(math.radians(30.0))
raw = torch.randint(0, 4096, (n, h, w), dtype=torch.int32, device="cuda").to(torch.uint16)
res = deskew_device(raw, s, "linear")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()


def call():
    deskew_device(raw, s, "linear", volume=res.volume, projections=res.projections, stream=side)


with torch.cuda.stream(side):
    for _ in range(3):
        call()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=side):
    call()
torch.cuda.synchronize()

for label, fn in (("direct", call), ("graph", g.replay), ("direct", call), ("graph", g.replay)):
    pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    with torch.cuda.stream(side):
        for a, b in pairs:
            flush.fill_(1)
            a.record(side)
            fn()
            b.record(side)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in pairs)
    print(label, "median ms", round(t[len(t) // 2], 4), "min", round(t[0], 4))
