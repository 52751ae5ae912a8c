"""Display encode, host side: oracle vs the reference's packets, header packing, errors.

Fixtures: tests/golden/display.npz (the reference's encode_frame_packet, ss/server.py:72-117).
"""
import struct

import numpy as np
import pytest

from ssb_testutil import display_cases  # noqa: F401  (also puts the repo on sys.path)

from oracle import deskew_oracle as O
from paper_2211_00645_b200 import display as D
from paper_2211_00645_b200.errors import ParameterError
from paper_2211_00645_b200.pipeline import DisplayImage, StageTimings

CASES = display_cases()


@pytest.mark.parametrize("k", range(len(CASES)))
def test_oracle_gray8_matches_reference_packet(k):
    img, _, pk = CASES[k]
    payload, off, rng = O.encode_gray8(img.pixels)
    g8_off, g8_rng = struct.unpack_from("<HH", pk["gray8"], 34)  # after 4sHBBHIIiIII
    assert (off, rng) == (g8_off, g8_rng)
    assert payload.tobytes() == pk["gray8"][64:]


@pytest.mark.parametrize("k", range(len(CASES)))
def test_header_matches_reference(k):
    img, tele, pk = CASES[k]
    assert D.frame_header(img, "gray16", 0, 0, tele) == pk["gray16"][:64]
    _, off, rng = O.encode_gray8(img.pixels)
    assert D.frame_header(img, "gray8", off, rng, tele) == pk["gray8"][:64]


@pytest.mark.parametrize("k", range(len(CASES)))
def test_gray16_packet_matches_reference(k):
    # gray16 is a byte copy of the image (no device work for a host image)
    img, tele, pk = CASES[k]
    assert D.encode_frame_packet(img, "gray16", tele) == pk["gray16"]


def test_wire_constants():
    assert D.HEADER_SIZE == 64
    assert D.PIXEL_FORMATS == {"gray16": 0, "gray8": 1}


def test_unknown_pixel_format():
    img = DisplayImage(pixels=np.zeros((2, 2), np.uint16), channel_id=0, sweep_index=0, slice_index=0,
                       view_angle_deg=30.0, mode="global", out_pitch_um=0.1, lateral_pitch_um=0.1)
    with pytest.raises(ParameterError, match="pixel format"):
        D.encode_frame_packet(img, "rgb")


def test_stage_timings_validation():
    with pytest.raises(ParameterError, match="lag_ms"):
        StageTimings(1.0, 1.0, 1.0, -1.0)
    assert StageTimings(1.0, 2.0, 3.0, 4.0).as_dict()["plotting_ms"] == 3.0
