"""Parity at BASELINE.json's sizes (configs 1 and 2) on the GPU.

Config 1 (128 x 256 x 512) is checked voxel for voxel against the C oracle; config 3
(200 x 1024 x 1024) through the pinned streaming pipeline against the oracle's projections.
Config 2 (512 x 2048 x 2048, the headline) is checked voxel for voxel against the C oracle
(in 64-slice chunks) and with size-independent
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
