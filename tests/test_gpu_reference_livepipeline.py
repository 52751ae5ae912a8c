"""The reference's ``LivePipeline`` (ss/pipeline.py:706-1064), unmodified, on the drop-in canvas.

Differential test: the same scripted acquisition -- random 16-bit frames, two channels split from
one camera frame, a view-angle change, a switch to rolling mode and back, a direct shear change --
runs twice through the reference's own ``LivePipeline.step()`` (``baseline/_ref``), once with its
numpy ``ProjectionCanvas`` / ``warp_projection`` and once with the drop-in's (canvas in HBM, fused
sm_100a kernels).  Every emitted ``DisplayImage`` must be identical: pixels bit for bit, plus sweep,
slice, channel, mode and view angle.  This exercises the paths the reference drives on a canvas:
``_ChannelState`` construction (:677-700), ``_apply_channel_params`` assigning ``canvas.mode`` /
``canvas.ring`` and calling ``replace_all`` (:851-871), ``place`` / ``finalize_global`` /
``rolling_replace`` and the rolling-mode ``canvas.max_pixels.copy()`` (:918-932).
"""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = os.path.join(REPO, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "skewstream")),
                                 reason="reference not installed (baseline/install_ref.sh)")]


def _ref_modules():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import skewstream.clock as rclock
    import skewstream.errors as rerrors
    import skewstream.geometry as rgeom
    import skewstream.pipeline as rpipe

    from paper_2211_00645_b200 import errors

    errors.adopt(rerrors)
    return rpipe, rgeom, rclock


class _Camera:
    """Scripted camera on a virtual clock: frame k of the acquisition is frames[k]."""

    def __init__(self, rpipe, clock, frames, n_slices, period_ns=5_000_000):
        self.rpipe, self.clock, self.frames, self.n = rpipe, clock, frames, n_slices
        self.period_ns, self.k = period_ns, 0

    def set_exposure_ms(self, ms):
        pass

    def next_frame(self):
        sweep, idx = divmod(self.k, self.n)
        px = self.frames[self.k]
        self.k += 1
        self.clock.sleep_until(self.clock.now_ns() + self.period_ns)
        return self.rpipe.RawFrame(pixels=px, slice_index=idx, sweep_index=sweep, channel_id=0,
                                   timestamp_ns=self.clock.now_ns())


def _run(rpipe, rgeom, rclock, canvas_cls, warp_fn, interp, frames, n, schedule, layout):
    saved = rpipe.ProjectionCanvas, rpipe.warp_projection
    rpipe.ProjectionCanvas, rpipe.warp_projection = canvas_cls, warp_fn
    try:
        h, w = frames.shape[1:]
        g = rgeom.SheetGeometry(alpha_deg=30.0, scan_step_um=0.115, pixel_pitch_um=0.115, slice_count=n,
                                frame_width_px=w, frame_height_px=h)
        clock = rclock.VirtualClock()
        cam = _Camera(rpipe, clock, frames, n)
        cfg = rpipe.PipelineConfig(geom=g, mode="global", interp=interp, layout=layout)
        pipe = rpipe.LivePipeline(cam, cfg, clock=clock)
        out = []
        for k in range(len(frames)):
            if k in schedule:
                pipe.post_params(**schedule[k])
            for im in pipe.step():
                out.append((np.array(im.pixels), im.channel_id, im.sweep_index, im.slice_index, im.mode,
                            round(im.view_angle_deg, 9)))
        return out
    finally:
        rpipe.ProjectionCanvas, rpipe.warp_projection = saved


@pytest.mark.parametrize("interp", ["linear", "nearest"])
def test_live_pipeline_emits_identical_images_on_drop_in(interp):
    rpipe, rgeom, rclock = _ref_modules()
    from paper_2211_00645_b200 import pipeline as dp

    n, h, w, sweeps = 12, 40, 96, 7
    frames = np.random.default_rng(11).integers(0, 65536, size=(sweeps * n, h, 2 * w), dtype=np.uint16)
    # two channels side by side on the camera (split_channels, ss/pipeline.py:105-112)
    layout = rpipe.ChannelLayout(regions=(rpipe.ChannelRegion(0, 0, 0, w, h), rpipe.ChannelRegion(1, w, 0, w, h)))
    schedule = {
        17: {"view_angle_deg": 40.0},      # lands at the next sweep start (global mode)
        30: {"mode": "rolling"},           # ring re-armed, replace_all at the frame boundary
        41: {"view_angle_deg": 25.0},      # rolling: replace_all under the new shear
        55: {"shear_px": 1.5},             # direct shear change
        63: {"mode": "global"},
    }
    ref = _run(rpipe, rgeom, rclock, rpipe.ProjectionCanvas, rpipe.warp_projection, interp, frames, n, schedule,
               layout)
    ours = _run(rpipe, rgeom, rclock, dp.ProjectionCanvas, dp.warp_projection, interp, frames, n, schedule, layout)
    assert len(ref) > 2 * sweeps  # global emissions plus one per frame while rolling
    assert len(ours) == len(ref)
    modes = {r[4] for r in ref}
    assert modes == {"global", "rolling"}
    for k, (a, b) in enumerate(zip(ref, ours)):
        assert a[1:] == b[1:], (k, a[1:], b[1:])
        assert a[0].shape == b[0].shape, (k, a[0].shape, b[0].shape)
        np.testing.assert_array_equal(b[0], a[0], err_msg=f"emission {k} {a[1:]}")
