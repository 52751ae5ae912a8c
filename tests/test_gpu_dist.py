"""Device half of the multi-GPU path on one GPU: every slab of a long scan deskewed by
the kernel over its own canvas window (global slice indices), merged on the host,
must equal the single-launch result.  (The collective half runs over gloo in
test_dist_cpu.py; kernels that wait on other ranks are never emulated on one GPU.)"""

import numpy as np
import pytest
import torch

from paper_2211_00645_b200 import dist as D
from paper_2211_00645_b200.deskew import deskew_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,halo", [(2, 0), (3, 0), (8, 0), (3, 2)])
@pytest.mark.parametrize("reduce", ["sum", "max"])
def test_slabs_merge_to_full_scan(world, halo, reduce):
    n, h, w, s = 300, 96, 512, 0.7071067811865476
    g = torch.Generator(device="cuda").manual_seed(world)
    raw = torch.randint(0, 65536, (n, h, w), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)
    full = deskew_device(raw, s, "linear", reduce=reduce, write_volume=False)
    plans = D.plan_slabs(n, h, s, "linear", world, halo=halo)
    U = plans[0].canvas_rows
    xy = torch.zeros((U, w), dtype=torch.int64, device="cuda")
    xz, yz = [], []
    for p in plans:
        part = D.deskew_slab(raw[p.in_first:p.in_first + p.in_count], p, s, "linear", reduce=reduce,
                             projection_axes=(0, 1, 2))
        win = part.projections[0].to(torch.int64)
        if reduce == "max":
            xy[p.u_begin:p.u_begin + p.u_count] = torch.maximum(xy[p.u_begin:p.u_begin + p.u_count], win)
        else:
            xy[p.u_begin:p.u_begin + p.u_count] += win
        xz.append(part.projections[1].to(torch.int64))
        row = torch.zeros((p.count, U), dtype=torch.int64, device="cuda")
        row[:, p.u_begin:p.u_begin + p.u_count] = part.projections[2].to(torch.int64)
        yz.append(row)
    torch.cuda.synchronize()
    assert torch.equal(xy, full.projections[0].to(torch.int64))
    assert torch.equal(torch.cat(xz), full.projections[1].to(torch.int64))
    assert torch.equal(torch.cat(yz), full.projections[2].to(torch.int64))


def test_config5_slab_window_runs():
    # one rank's share of the config-5 scan (1024 of 8192 frames, 45 deg), projection-only sum
    plans = D.plan_slabs(8192, 2048, 0.7071067811865476, "linear", 8)
    p = plans[3]
    g = torch.Generator(device="cuda").manual_seed(5)
    raw = torch.randint(0, 4096, (p.count, 2048, 2048), generator=g, device="cuda",
                        dtype=torch.int32).to(torch.uint16)
    res = D.deskew_slab(raw, p, 0.7071067811865476, "linear", reduce="sum", projection_axes=(0,))
    torch.cuda.synchronize()
    xy = res.projections[0]
    assert tuple(xy.shape) == (p.u_count, 2048)
    assert xy.dtype == torch.uint32
    # linearity of the sum projection: the slab's XY equals the sum of its two halves' XY,
    # each deskewed over its own canvas window with global slice indices
    half = p.count // 2
    acc = torch.zeros((p.u_count, 2048), dtype=torch.int64, device="cuda")
    for first, count in ((p.first, half), (p.first + half, p.count - half)):
        sub = D.SlabPlan(p.rank, first, count, p.u_begin, p.u_count, p.canvas_rows)
        r = D.deskew_slab(raw[first - p.first:first - p.first + count], sub, 0.7071067811865476, "linear",
                          reduce="sum", projection_axes=(0,))
        acc += r.projections[0].to(torch.int64)
    torch.cuda.synchronize()
    assert torch.equal(acc, xy.to(torch.int64))
    assert int(acc.sum()) > 0


def test_config5_slab_sum_matches_oracle():
    """Config 5 semantics against the C oracle: 64 frames from the middle of the 8192-frame scan
    (45 deg, global slice indices), XY sum (uint32) over the owning rank's canvas row window."""
    from oracle import c_oracle as C

    s45 = 0.7071067811865476
    p = D.plan_slabs(8192, 2048, s45, "linear", 8)[5]
    first, count = p.first + 480, 64
    g = torch.Generator(device="cuda").manual_seed(55)
    raw = torch.randint(0, 65536, (count, 2048, 2048), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)
    sub = D.SlabPlan(p.rank, first, count, p.u_begin, p.u_count, p.canvas_rows)
    res = D.deskew_slab(raw, sub, s45, "linear", reduce="sum", projection_axes=(0,))
    torch.cuda.synchronize()
    _, want = C.deskew(raw.cpu().numpy(), s45, "linear", reduce="sum", first_slice=first, u_begin=p.u_begin,
                       u_count=p.u_count, want_volume=False, axes=(0,))
    np.testing.assert_array_equal(res.projections[0].cpu().numpy(), want[0])
