"""Display encode on the GPU (ssb_encode_gray8) against the reference's packets and the oracle."""
import numpy as np
import pytest
import torch

from ssb_testutil import display_cases

from oracle import deskew_oracle as O
from paper_2211_00645_b200 import _lib
from paper_2211_00645_b200 import display as D
from paper_2211_00645_b200.pipeline import DisplayImage

pytestmark = pytest.mark.gpu
CASES = display_cases()


@pytest.mark.parametrize("k", range(len(CASES)))
@pytest.mark.parametrize("fmt", ["gray8", "gray16"])
def test_packet_matches_reference(k, fmt):
    img, tele, pk = CASES[k]
    n0 = _lib.launch_count()
    assert D.encode_frame_packet(img, fmt, tele) == pk[fmt]
    if fmt == "gray8":
        assert _lib.launch_count() - n0 == 1  # one cooperative launch


@pytest.mark.parametrize("k", range(len(CASES)))
def test_device_image_input(k):
    img, tele, pk = CASES[k]
    dev = torch.from_numpy(img.pixels.view(np.int16)).cuda().view(torch.uint16)
    dimg = DisplayImage(pixels=dev, channel_id=img.channel_id, sweep_index=img.sweep_index,
                        slice_index=img.slice_index, view_angle_deg=img.view_angle_deg, mode=img.mode,
                        out_pitch_um=img.out_pitch_um, lateral_pitch_um=img.lateral_pitch_um,
                        timings=img.timings)
    assert D.encode_frame_packet(dimg, "gray8", tele) == pk["gray8"]
    assert D.encode_frame_packet(dimg, "gray16", tele) == pk["gray16"]


@pytest.mark.parametrize("shape,hi,misalign", [((2491, 2048), 65536, 0), ((1197, 1024), 4096, 0),
                                               ((777, 1001), 65536, 1), ((1, 9), 3, 1),
                                               ((5000, 3), 65536, 3)])
def test_large_and_misaligned_against_oracle(shape, hi, misalign):
    rng = np.random.default_rng(shape[0])
    n = shape[0] * shape[1]
    flat = rng.integers(0, hi, n + misalign).astype(np.uint16)
    dev = torch.from_numpy(flat.view(np.int16)).cuda().view(torch.uint16)
    img = dev[misalign:].view(shape)  # odd element offset -> scalar path
    payload, stats = D.encode_gray8_device(img)
    ref, off, rg = O.encode_gray8(flat[misalign:].reshape(shape))
    assert np.array_equal(payload.cpu().numpy(), ref)
    assert [int(v) for v in stats[:2].cpu()] == [off, rg]


def test_constant_and_two_level_images():
    for px in (np.full((64, 64), 7, np.uint16), np.zeros((3, 5), np.uint16),
               np.array([[0, 65535] * 8], np.uint16)):
        payload, stats = D.encode_gray8_device(px)
        ref, off, rg = O.encode_gray8(px)
        assert np.array_equal(payload.cpu().numpy(), ref)
        assert [int(v) for v in stats[:2].cpu()] == [off, rg]


def test_empty_image_raises_like_numpy():
    with pytest.raises(ValueError):
        D.encode_gray8_device(np.zeros((0, 4), np.uint16))


def test_stream_ordering_back_to_back():
    # two encodes on one stream reuse the stats buffer; results must not interfere
    a = torch.randint(0, 65536, (512, 512), dtype=torch.int32, device="cuda").to(torch.uint16)
    b = torch.randint(100, 200, (512, 512), dtype=torch.int32, device="cuda").to(torch.uint16)
    pa, _ = D.encode_gray8_device(a)
    pa = pa.clone()
    pb, sb = D.encode_gray8_device(b)
    ra, _, _ = O.encode_gray8(a.view(torch.int16).cpu().numpy().view(np.uint16))
    rb, off, rg = O.encode_gray8(b.view(torch.int16).cpu().numpy().view(np.uint16))
    assert np.array_equal(pa.cpu().numpy(), ra)
    assert np.array_equal(pb.cpu().numpy(), rb)
    assert [int(v) for v in sb[:2].cpu()] == [off, rg]
