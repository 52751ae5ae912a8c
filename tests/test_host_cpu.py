"""Host-side contract of the drop-in that runs without a GPU: frame/channel types,
argument validation (same exceptions and messages as the reference) and the
no-fallback rule (compute entry points raise instead of running on the CPU)."""

import numpy as np
import pytest
import torch

from paper_2211_00645_b200 import pipeline as pl
from paper_2211_00645_b200.errors import (CapacityError, DeviceError, ParameterError,
                                          SkewstreamError)
from ssb_testutil import geom

NO_GPU = not torch.cuda.is_available()


def frame(arr, i, **kw):
    return pl.RawFrame(np.asarray(arr, dtype=np.uint16), i, **kw)


class TestRawFrame:  # pkg/tests/test_pipeline.py:44-61
    def test_requires_uint16(self):
        with pytest.raises(ParameterError):
            pl.RawFrame(np.zeros((2, 2), np.float32), 0)

    def test_requires_2d(self):
        with pytest.raises(ParameterError):
            pl.RawFrame(np.zeros((2, 2, 2), np.uint16), 0)

    def test_negative_slice(self):
        with pytest.raises(ParameterError):
            pl.RawFrame(np.zeros((2, 2), np.uint16), -1)

    def test_shape(self):
        f = frame(np.zeros((3, 5)), 0)
        assert (f.height, f.width) == (3, 5)


class TestChannels:  # pkg/tests/test_pipeline.py:64-103
    def test_overlap_rejected(self):
        with pytest.raises(ParameterError, match="overlap"):
            pl.ChannelLayout(regions=(pl.ChannelRegion(0, 0, 0, 4, 4), pl.ChannelRegion(1, 2, 0, 4, 4)))

    def test_split_two_channels(self):
        layout = pl.ChannelLayout(regions=(pl.ChannelRegion(0, 0, 0, 2, 2), pl.ChannelRegion(1, 2, 0, 2, 2)))
        f = frame([[1, 2, 3, 4], [5, 6, 7, 8]], 3, sweep_index=1)
        subs = pl.split_channels(f, layout)
        assert [s.channel_id for s in subs] == [0, 1]
        np.testing.assert_array_equal(subs[0].pixels, [[1, 2], [5, 6]])
        np.testing.assert_array_equal(subs[1].pixels, [[3, 4], [7, 8]])
        subs[0].pixels[0, 0] = 99
        assert f.pixels[0, 0] == 1

    def test_region_exceeding_frame(self):
        with pytest.raises(ParameterError):
            pl.ChannelLayout(regions=(pl.ChannelRegion(0, 0, 0, 8, 8),)).validate_frame(4, 4)


class TestValidationBeforeDevice:
    def test_bad_interp_and_mode(self):  # pkg/tests/test_pipeline.py:216-222
        with pytest.raises(ParameterError):
            pl.ProjectionCanvas(geom(), 1.0, interp="cubic")
        with pytest.raises(ParameterError):
            pl.ProjectionCanvas(geom(), 1.0, mode="windowed")

    def test_canvas_limit(self):
        with pytest.raises(CapacityError):
            pl.ProjectionCanvas(geom(n=100_000, w=10_000, h=10_000), 1.0)

    def test_warp_bad_scale(self):  # pkg/tests/test_pipeline.py:296-302
        proj = np.zeros((4, 2), np.uint16)
        with pytest.raises(ParameterError):
            pl.warp_projection(proj, 0.0)
        with pytest.raises(ParameterError):
            pl.warp_projection(proj, -1.0)

    def test_reference_deskew_validation(self):  # pkg/tests/test_phantom.py:255-263
        from paper_2211_00645_b200 import phantom as ph
        with pytest.raises(ParameterError, match="frame 1"):
            ph.reference_deskew([np.zeros((2, 2), np.uint16), np.zeros((3, 2), np.uint16)], geom(), 1.0)
        with pytest.raises(ParameterError):
            ph.reference_deskew([np.zeros((2, 2), np.uint16)], geom(), 1.0, interp="cubic")
        with pytest.raises(ParameterError, match="empty"):
            ph.reference_deskew([], geom(), 1.0)

    def test_error_hierarchy(self):
        assert issubclass(DeviceError, SkewstreamError)
        assert issubclass(ParameterError, ValueError)


@pytest.mark.skipif(not NO_GPU, reason="checks the no-fallback rule on a CPU-only host")
class TestNoCpuFallback:
    def test_canvas_needs_device(self):
        with pytest.raises(DeviceError):
            pl.ProjectionCanvas(geom(), 1.0)

    def test_deskew_volume_needs_device(self):
        from paper_2211_00645_b200.deskew import deskew_volume
        with pytest.raises(DeviceError):
            deskew_volume(np.zeros((2, 4, 8), np.uint16), geom(n=2, w=8, h=4), 1.0)

    def test_deskew_device_rejects_host_tensor(self):
        from paper_2211_00645_b200.deskew import deskew_device
        with pytest.raises(ParameterError):
            deskew_device(torch.zeros((2, 4, 8), dtype=torch.uint16), 1.0)

    def test_batch_views_need_device(self):
        from paper_2211_00645_b200.batch import deskew_views
        from paper_2211_00645_b200.geometry import view_transform
        g = geom(n=2, w=8, h=4)
        with pytest.raises(DeviceError):
            deskew_views(np.zeros((2, 4, 8), np.uint16), g, [view_transform(g, view_angle_deg=30.0)])

    def test_warp_needs_device(self):
        with pytest.raises(DeviceError):
            pl.warp_projection(np.zeros((4, 2), np.uint16), 1.5)


class TestChunkBounds:
    """Chunking of the pinned H2D pipeline: full chunks, then a short last chunk (latency)."""

    def test_cover_in_order(self):
        from paper_2211_00645_b200.stream import chunk_bounds
        for n in (1, 7, 8, 9, 31, 32, 33, 200):
            for chunk in (1, 4, 32):
                for tail in (1, 2, 8):
                    b = chunk_bounds(n, chunk, min(tail, chunk))
                    assert b[0][0] == 0 and b[-1][1] == n
                    assert all(c1 > c0 for c0, c1 in b)
                    assert all(b[k][1] == b[k + 1][0] for k in range(len(b) - 1))
                    assert max(c1 - c0 for c0, c1 in b) <= chunk
                    assert b[-1][1] - b[-1][0] <= min(tail, chunk)

    def test_config3_shape(self):
        from paper_2211_00645_b200.stream import chunk_bounds
        # 200 frames of 1024^2: 64 MB chunks (32 frames), <= 16 MB (8 frames) last
        b = chunk_bounds(200, 32, 8)
        assert b[-1] == (192, 200) and len(b) == 7
        b = chunk_bounds(64, 32, 8)
        assert b == [(0, 32), (32, 56), (56, 64)]


class TestWorkspaceCache:
    def test_lru_bound(self):
        """Scratch buffers are kept per stream, least recently used evicted (CPU stand-in streams)."""
        from paper_2211_00645_b200.deskew import _Workspaces

        class FakeStream:
            def __init__(self, h):
                self.cuda_stream = h
                self.device = torch.device("cpu")

        ws = _Workspaces(max_streams=3)
        import contextlib
        orig = torch.cuda.stream
        torch.cuda.stream = lambda s: contextlib.nullcontext()
        try:
            bufs = [ws.get(1000, FakeStream(h)) for h in range(5)]
            assert len(ws._bufs) == 3
            assert ws.get(10, FakeStream(4)) is bufs[4]  # recent entry reused
            assert ws.get(10, FakeStream(0)) is not bufs[0]  # evicted entry re-created
        finally:
            torch.cuda.stream = orig


class TestHostView:
    """ProjectionCanvas.max_pixels / contributor host copies (pipeline._HostView): in-place writes
    mark the canvas dirty so the device copy is refreshed before its next operation."""

    class Owner:
        _host_dirty = False

    def make(self):
        from paper_2211_00645_b200.pipeline import _HostView

        o = self.Owner()
        v = np.zeros((4, 3), dtype=np.uint16).view(_HostView)
        v._owner = o
        return o, v

    def test_item_and_view_writes_mark_dirty(self):
        o, v = self.make()
        _ = v[1:3].sum(), v.max()  # reads do not
        assert not o._host_dirty
        v[1, 2] = 7
        assert o._host_dirty and v[1, 2] == 7
        o._host_dirty = False
        v[2:][0, 0] = 3  # through a view
        assert o._host_dirty

    def test_ufunc_out_marks_dirty_but_copies_do_not(self):
        o, v = self.make()
        np.maximum(v[0:2], 9, out=v[0:2])  # the reference's place() idiom (ss/pipeline.py:321)
        assert o._host_dirty and int(v[:2].min()) == 9
        o._host_dirty = False
        c = v.copy()
        c[0, 0] = 1
        a = np.array(v)
        a[0, 0] = 2
        assert not o._host_dirty and v[0, 0] == 9


def test_errors_adopt_reference_classes():
    """errors.adopt(skewstream.errors): the reference's except clauses catch the drop-in's errors."""
    import os
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "skewstream")):
        pytest.skip("reference not installed (baseline/install_ref.sh)")
    sys.path.insert(0, ref)
    import skewstream.errors as R

    from paper_2211_00645_b200 import errors as E

    E.adopt(R)
    E.adopt(R)  # idempotent
    for name in E._CLASSES:
        assert issubclass(getattr(E, name), getattr(R, name)), name
    assert issubclass(E.ParameterError, ValueError)
    assert issubclass(E.DeviceError, R.SkewstreamError)
    with pytest.raises(R.CapacityError):
        raise E.CapacityError("span outside canvas")
