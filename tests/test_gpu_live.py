"""Live-view channel driver (live.ChannelDeskewer) replaying the reference LivePipeline.

tests/golden/live.npz holds, per scenario, the scripted frames, the parameter changes and the
DisplayImages the reference's LivePipeline.step emitted (ss/pipeline.py:850-980).
"""
import os

import numpy as np
import pytest
import torch

from ssb_testutil import GOLDEN, geom

from paper_2211_00645_b200 import display as D
from paper_2211_00645_b200.geometry import ViewTransform
from paper_2211_00645_b200.live import ChannelDeskewer
from paper_2211_00645_b200.pipeline import RawFrame

pytestmark = pytest.mark.gpu
LIVE = dict(np.load(os.path.join(GOLDEN, "live.npz")))
MODES = ["global", "rolling"]


def replay(k, device_pixels=False):
    n, h, w, _ = (int(v) for v in LIVE[f"s{k}_meta"])
    g = geom(n=n, h=h, w=w, alpha=60.0, step=0.2, pitch=0.1)
    ch = ChannelDeskewer(0, g, ViewTransform(*LIVE[f"s{k}_vt0"]), str(LIVE[f"s{k}_interp"]),
                         str(LIVE[f"s{k}_mode"]), device_pixels=device_pixels)
    changes = {int(c[0]): (int(c[1]), int(c[2]), vt) for c, vt in zip(LIVE[f"s{k}_changes"], LIVE[f"s{k}_change_vt"])}
    out = []
    for step, (px, (sweep, idx)) in enumerate(zip(LIVE[f"s{k}_frames"], LIVE[f"s{k}_frame_ids"])):
        if step in changes:
            kind, mode, vt = changes[step]
            if kind == 2:
                ch.set_mode(MODES[mode])
            else:
                ch.set_view(ViewTransform(*vt))
        im = ch.process(RawFrame(px, int(idx), int(sweep), 0, timestamp_ns=7_000_000 * (step + 1)))
        if im is not None:
            out.append((step, im))
    return out


@pytest.mark.parametrize("k", range(int(LIVE["count"])))
def test_emissions_match_reference_live_pipeline(k):
    got = replay(k)
    assert len(got) == int(LIVE[f"s{k}_emit_count"])
    for e, (step, im) in enumerate(got):
        ref_step, sweep, sl, mode = (int(v) for v in LIVE[f"s{k}_e{e}_ids"])
        angle, pitch, lateral, acq = LIVE[f"s{k}_e{e}_f"]
        assert (step, im.sweep_index, im.slice_index, im.mode) == (ref_step, sweep, sl, MODES[mode])
        np.testing.assert_array_equal(im.pixels, LIVE[f"s{k}_e{e}_px"])
        assert im.view_angle_deg == angle and im.out_pitch_um == pitch and im.lateral_pitch_um == lateral
        assert im.timings.acquisition_ms == pytest.approx(acq)
        assert im.timings.processing_ms > 0 and im.timings.plotting_ms >= 0


def test_device_pixels_feed_the_display_encoder():
    got = replay(0, device_pixels=True)
    assert got and all(isinstance(im.pixels, torch.Tensor) and im.pixels.is_cuda for _, im in got)
    pkt = D.encode_frame_packet(got[-1][1], "gray8")
    host = type(got[-1][1])(**{**got[-1][1].__dict__, "pixels": got[-1][1].pixels.cpu().numpy().view(np.uint16)})
    assert pkt[64:] == D.encode_frame_packet(host, "gray8")[64:]
