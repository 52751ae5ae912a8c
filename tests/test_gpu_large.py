"""Parity at BASELINE.json's sizes (configs 1 and 2) on the GPU.

Config 1 (128 x 256 x 512) is checked voxel for voxel against the C oracle; config 3
(200 x 1024 x 1024) through the pinned streaming pipeline against the oracle's projections.
Config 2 (512 x 2048 x 2048, the headline) is checked voxel for voxel against the C oracle
(in 64-slice chunks; also at W = 2044 / 2047, the row-class TMA mode) and with size-independent
properties: sampled slices against the oracle (global slice index, full canvas
row window), every projection against a reduction of the kernel's own volume,
and the XY canvas against the oracle's streaming canvas.
"""

import numpy as np
import pytest
import torch

from oracle import c_oracle as C
from paper_2211_00645_b200.deskew import deskew_device

pytestmark = pytest.mark.gpu
S30 = 0.8660254037844386  # native shear at 30 degrees, step == pitch


def synthetic(n, h, w, seed, hi=4096):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randint(0, hi, (n, h, w), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)


@pytest.fixture(params=["tma", "tiled"])
def kernel_path(request, monkeypatch):
    if request.param == "tiled":
        monkeypatch.setenv("SSB_DISABLE_TMA", "1")
    else:
        monkeypatch.delenv("SSB_DISABLE_TMA", raising=False)
    return request.param


@pytest.mark.parametrize("interp", ["linear", "nearest"])
@pytest.mark.parametrize("reduce", ["max", "sum"])
def test_config1_full_parity(interp, reduce, kernel_path):
    raw = synthetic(128, 256, 512, 1, hi=65536)
    res = deskew_device(raw, S30, interp, reduce=reduce)
    torch.cuda.synchronize()
    st = raw.cpu().numpy()
    want_vol, want = C.deskew(st, S30, interp, reduce=reduce)
    assert res.volume.shape == (128, 366, 512)
    np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
    for ax in (0, 1, 2):
        np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])


def _reduce_dev(vol: torch.Tensor, axis: int, reduce: str) -> np.ndarray:
    out = None
    step = 64
    if axis == 0:
        for k in range(0, vol.shape[0], step):
            part = vol[k:k + step].to(torch.int32)
            r = part.amax(0) if reduce == "max" else part.sum(0, dtype=torch.int64)
            out = r if out is None else (torch.maximum(out, r) if reduce == "max" else out + r)
        return out.cpu().numpy()
    parts = []
    for k in range(0, vol.shape[0], step):
        part = vol[k:k + step].to(torch.int32)
        parts.append((part.amax(axis) if reduce == "max" else part.sum(axis, dtype=torch.int64)).cpu())
    return torch.cat(parts).numpy()


@pytest.mark.parametrize("reduce", ["max", "sum"])
def test_config2_properties(reduce, kernel_path):
    n, h, w = 512, 2048, 2048
    raw = synthetic(n, h, w, 2)
    res = deskew_device(raw, S30, "linear", reduce=reduce)
    torch.cuda.synchronize()
    assert res.volume.shape == (n, 2491, w)
    # projections == reductions of the kernel's own volume
    for ax in (0, 1, 2):
        got = res.projections[ax].cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(got, _reduce_dev(res.volume, ax, reduce).astype(np.int64))
    # sampled slices vs the oracle, global index, full canvas window
    for k in (0, 1, 173, 510, 511):
        st = raw[k:k + 1].cpu().numpy()
        want_vol, _ = C.deskew(st, S30, "linear", first_slice=k, u_begin=0, u_count=2491, axes=())
        np.testing.assert_array_equal(res.volume[k:k + 1].cpu().numpy(), want_vol)
    if reduce == "max":
        # the reference's own product: the streaming canvas
        _, want = C.deskew(raw.cpu().numpy(), S30, "linear", want_volume=False, axes=(0,))
        np.testing.assert_array_equal(res.projections[0].cpu().numpy(), want[0])


def test_config2_projection_only_matches_volume_path():
    raw = synthetic(512, 2048, 2048, 3)
    full = deskew_device(raw, S30, "linear")
    proj = deskew_device(raw, S30, "linear", write_volume=False)
    torch.cuda.synchronize()
    for ax in (0, 1, 2):
        assert torch.equal(full.projections[ax].view(torch.int16), proj.projections[ax].view(torch.int16))


@pytest.mark.parametrize("interp", ["linear", "nearest"])
def test_config2_full_volume_voxel_for_voxel(interp):
    """The headline workload checked voxel for voxel: all 512 deskewed slices of a 512 x 2048 x 2048
    stack (full 16-bit range) against the C oracle, in 64-slice chunks with global slice indices,
    plus every projection against the oracle's."""
    n, h, w, U = 512, 2048, 2048, 2491
    raw = synthetic(n, h, w, 5, hi=65536)
    res = deskew_device(raw, S30, interp, reduce="max")
    torch.cuda.synchronize()
    assert res.volume.shape == (n, U, w)
    xy = np.zeros((U, w), np.uint16)
    for k in range(0, n, 64):
        st = raw[k:k + 64].cpu().numpy()
        want_vol, want = C.deskew(st, S30, interp, first_slice=k, u_begin=0, u_count=U)
        np.testing.assert_array_equal(res.volume[k:k + 64].cpu().numpy(), want_vol, err_msg=f"slices {k}..{k + 63}")
        np.testing.assert_array_equal(res.projections[1][k:k + 64].cpu().numpy(), want[1])
        np.testing.assert_array_equal(res.projections[2][k:k + 64].cpu().numpy(), want[2])
        np.maximum(xy, want[0], out=xy)
    np.testing.assert_array_equal(res.projections[0].cpu().numpy(), xy)


@pytest.mark.parametrize("interp,w", [("linear", 2044), ("nearest", 2044), ("linear", 2047)])
def test_config2_odd_width_voxel_for_voxel(interp, w):
    """Config 2's shape with rows that are not 16-byte aligned (W = 2044: 8-byte rows, two row classes;
    W = 2047: 2-byte rows, eight classes) through the row-class TMA mode: every slice against the C
    oracle (64-slice chunks, global indices), every projection too."""
    n, h, U = 512, 2048, 2491
    raw = synthetic(n, h, w, 7, hi=65536)
    res = deskew_device(raw, S30, interp, reduce="max")
    torch.cuda.synchronize()
    assert res.volume.shape == (n, U, w)
    xy = np.zeros((U, w), np.uint16)
    for k in range(0, n, 64):
        st = raw[k:k + 64].cpu().numpy()
        want_vol, want = C.deskew(st, S30, interp, first_slice=k, u_begin=0, u_count=U)
        np.testing.assert_array_equal(res.volume[k:k + 64].cpu().numpy(), want_vol, err_msg=f"slices {k}..{k + 63}")
        np.testing.assert_array_equal(res.projections[1][k:k + 64].cpu().numpy(), want[1])
        np.testing.assert_array_equal(res.projections[2][k:k + 64].cpu().numpy(), want[2])
        np.maximum(xy, want[0], out=xy)
    np.testing.assert_array_equal(res.projections[0].cpu().numpy(), xy)


def test_config3_live_stream_matches_oracle():
    """Config 3 as bench.py streams it: 200 x 1024 x 1024 from pinned host memory through the
    chunked H2D pipeline (64 MB chunks, short last chunk), projection-only XY/XZ/YZ max, against
    the C oracle's projections."""
    from paper_2211_00645_b200.stream import StackStreamer, pinned_stack

    n, h, w = 200, 1024, 1024
    host = pinned_stack(n, h, w)
    host[:] = np.random.default_rng(33).integers(0, 65536, (n, h, w), dtype=np.uint16)
    streamer = StackStreamer(h, w)
    assert streamer.chunk_bounds(n)[-1][1] - streamer.chunk_bounds(n)[-1][0] <= streamer.tail
    res = streamer.run(host, S30, "linear", reduce="max", write_volume=False)
    torch.cuda.synchronize()
    _, want = C.deskew(np.asarray(host), S30, "linear", want_volume=False)
    for ax in (0, 1, 2):
        np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])


def test_config5_full_scan_sum_matches_oracle():
    """Config 5 at full size: 8192 x 2048 x 2048 frames (68.7 GB, resident), 45 degrees, XY sum.

    One projection-only launch over the whole scan, and the 8-slab split (dist.plan_slabs, global
    slice indices, per-slab canvas row windows) merged on the device, are both compared with the C
    oracle run chunk by chunk (512 frames, global indices) and accumulated in uint64 on the host.
    Full 16-bit range, so the fp32 bracket's fallback and the per-tile slice-range clipping
    (ssb_tma_kernel.cuh tile_slices) are exercised where a long scan stresses them most.
    """
    from paper_2211_00645_b200 import dist as D
    from paper_2211_00645_b200.deskew import canvas_rows_for

    n, h, w, s45, chunk = 8192, 2048, 2048, 0.7071067811865476, 512
    U = canvas_rows_for(n, h, s45)
    raw = torch.empty((n, h, w), dtype=torch.uint16, device="cuda")
    for c0 in range(0, n, chunk):
        g = torch.Generator(device="cuda").manual_seed(5000 + c0)
        raw[c0:c0 + chunk] = torch.randint(0, 65536, (chunk, h, w), generator=g, device="cuda",
                                           dtype=torch.int32).to(torch.uint16)
    full = deskew_device(raw, s45, "linear", reduce="sum", projection_axes=(0,), write_volume=False)
    slabs = torch.zeros((U, w), dtype=torch.int64, device="cuda")
    for p in D.plan_slabs(n, h, s45, "linear", 8):
        part = D.deskew_slab(raw[p.first:p.first + p.count], p, s45, "linear", reduce="sum", projection_axes=(0,))
        slabs[p.u_begin:p.u_begin + p.u_count] += part.projections[0].to(torch.int64)
    got_full = full.projections[0].to(torch.int64).cpu().numpy()
    got_slabs = slabs.cpu().numpy()
    assert got_full.shape == (U, w)

    want = np.zeros((U, w), dtype=np.uint64)
    host = torch.empty((chunk, h, w), dtype=torch.uint16, pin_memory=True)
    for c0 in range(0, n, chunk):
        host.copy_(raw[c0:c0 + chunk])
        plan = D.plan_slabs(chunk, h, s45, "linear", 1)[0]  # canvas row window of frames c0..c0+chunk
        lo = int(np.ceil(c0 * s45 - 1e-9))
        hi = min(U - 1, lo + plan.u_count + 2)
        _, o = C.deskew(host.numpy(), s45, "linear", reduce="sum", first_slice=c0, u_begin=lo,
                        u_count=hi - lo + 1, want_volume=False, axes=(0,))
        want[lo:hi + 1] += o[0]
    del raw
    np.testing.assert_array_equal(got_full, want.astype(np.int64))
    np.testing.assert_array_equal(got_slabs, want.astype(np.int64))
