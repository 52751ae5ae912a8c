"""Small driver for ncu captures: config-2 fused deskew launches, nothing else."""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00645_b200.deskew import deskew_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--interp", default="linear")
ap.add_argument("--reduce", default="max")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--hw", type=int, default=2048)
ap.add_argument("--h", type=int, default=0, help="frame rows (default: --hw)")
ap.add_argument("--w", type=int, default=0, help="frame columns (default: --hw)")
ap.add_argument("--no-volume", action="store_true")
ap.add_argument("--formula", default="canvas")
ap.add_argument("--axes", default="0,1,2")
ap.add_argument("--alpha", type=float, default=30.0)
ap.add_argument("--batch", type=int, default=0, help="B > 0: deskew_batch over B distinct stacks")
a = ap.parse_args()
axes = tuple(int(v) for v in a.axes.split(","))
s = math.cos(math.radians(a.alpha))
g = torch.Generator(device="cuda").manual_seed(1234)
fh, fw = a.h or a.hw, a.w or a.hw
raw = torch.randint(0, 4096, (a.n, fh, fw), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)
if a.batch:
    from paper_2211_00645_b200.deskew import deskew_batch

    stacks = torch.stack([((raw.to(torch.int32) + 37 * k) % 4096).to(torch.uint16) for k in range(a.batch)])
    r = deskew_batch(stacks, s, a.interp, reduce=a.reduce, formula=a.formula, write_volume=not a.no_volume,
                     projection_axes=axes)
    for _ in range(a.iters):
        deskew_batch(stacks, s, a.interp, reduce=a.reduce, formula=a.formula, write_volume=not a.no_volume,
                     projection_axes=axes, volume=r.volume, projections=r.projections)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        deskew_batch(stacks, s, a.interp, reduce=a.reduce, formula=a.formula, write_volume=not a.no_volume,
                     projection_axes=axes, volume=r.volume, projections=r.projections)
    e1.record()
    torch.cuda.synchronize()
    print(f"batch {a.batch} {a.interp} {a.reduce} vol={not a.no_volume} axes={a.axes}: "
          f"{e0.elapsed_time(e1) / a.iters:.4f} ms/call")
    sys.exit(0)
res = None
for _ in range(a.iters):
    res = deskew_device(raw, s, a.interp, reduce=a.reduce, formula=a.formula, write_volume=not a.no_volume,
                        projection_axes=axes)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    deskew_device(raw, s, a.interp, reduce=a.reduce, formula=a.formula, write_volume=not a.no_volume,
                  volume=res.volume, projections=res.projections, projection_axes=axes)
e1.record()
torch.cuda.synchronize()
print(f"{a.interp} {a.reduce} vol={not a.no_volume} axes={a.axes}: {e0.elapsed_time(e1) / a.iters:.3f} ms/call")
