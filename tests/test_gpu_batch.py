"""Batched launches (``ssb_deskew_batch`` / ``deskew.deskew_batch``): B stacks in one persistent
launch give, stack by stack, exactly what one ``ssb_deskew`` per stack gives -- and, for config 1's
shape, what the C oracle gives."""

import numpy as np
import pytest
import torch

from oracle import c_oracle as C
from paper_2211_00645_b200.deskew import deskew_batch, deskew_device
from paper_2211_00645_b200.errors import ParameterError

pytestmark = pytest.mark.gpu
S30 = 0.8660254037844386


def stacks(b, n, h, w, seed, hi=65536):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randint(0, hi, (b, n, h, w), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)


@pytest.mark.parametrize("interp", ["linear", "nearest"])
@pytest.mark.parametrize("reduce", ["max", "sum"])
@pytest.mark.parametrize("formula", ["canvas", "npinterp"])
def test_batch_equals_per_stack(interp, reduce, formula):
    raw = stacks(5, 37, 48, 264, 7)
    s = 0.7
    got = deskew_batch(raw, s, interp, formula=formula, reduce=reduce)
    for k in range(raw.shape[0]):
        one = deskew_device(raw[k], s, interp, formula=formula, reduce=reduce)
        assert torch.equal(got.volume[k], one.volume), k
        for a in (0, 1, 2):
            assert torch.equal(got.projections[a][k], one.projections[a]), (k, a)


@pytest.mark.parametrize("axes,volume", [((0,), False), ((0, 1, 2), False), ((1,), True), ((0, 2), True)])
def test_batch_output_subsets(axes, volume):
    raw = stacks(3, 64, 96, 512, 3, hi=4096)
    got = deskew_batch(raw, S30, "linear", projection_axes=axes, write_volume=volume)
    assert (got.volume is not None) == volume
    for k in range(3):
        one = deskew_device(raw[k], S30, "linear", projection_axes=axes, write_volume=volume)
        if volume:
            assert torch.equal(got.volume[k], one.volume)
        for a in axes:
            assert torch.equal(got.projections[a][k], one.projections[a]), (k, a)


def test_config1_batch_of_16_matches_oracle():
    # BASELINE config 1 shape (128 x 256 x 512, 30 deg), 16 distinct stacks in one launch
    raw = stacks(16, 128, 256, 512, 16)
    got = deskew_batch(raw, S30, "linear")
    torch.cuda.synchronize()
    for k in (0, 7, 15):
        vol, pr = C.deskew(raw[k].cpu().numpy(), S30, "linear")
        np.testing.assert_array_equal(got.volume[k].cpu().numpy(), vol)
        for a in (0, 1, 2):
            np.testing.assert_array_equal(got.projections[a][k].cpu().numpy(), pr[a])


def test_unaligned_width_falls_back_stack_by_stack():
    raw = stacks(3, 20, 32, 203, 5)  # W % 8 != 0: no TMA boxes, one launch per stack
    got = deskew_batch(raw, 1.3, "linear", reduce="sum")
    for k in range(3):
        one = deskew_device(raw[k], 1.3, "linear", reduce="sum")
        assert torch.equal(got.volume[k], one.volume)
        for a in (0, 1, 2):
            assert torch.equal(got.projections[a][k], one.projections[a])


def test_batch_rejects_bad_input():
    with pytest.raises(ParameterError):
        deskew_batch(stacks(1, 4, 8, 16, 1)[0], 1.0)  # 3-D
    with pytest.raises(ParameterError):
        deskew_batch(stacks(2, 4, 8, 16, 1), -1.0)
