"""CUDA parity: libssb kernels (through the C ABI) vs the oracle and the reference's
own fixtures and hand examples.  Integer output => bit-exact everywhere."""

import os

import numpy as np
import pytest
import torch

from oracle import c_oracle as C
from oracle import deskew_oracle as O
from paper_2211_00645_b200 import _lib
from paper_2211_00645_b200 import phantom as ph
from paper_2211_00645_b200 import pipeline as pl
from paper_2211_00645_b200.deskew import deskew_device, deskew_volume
from paper_2211_00645_b200.errors import CapacityError, ParameterError, ProtocolError
from ssb_testutil import GOLDEN, geom, golden_cases

pytestmark = pytest.mark.gpu
CASES = golden_cases()


def dev():
    assert torch.cuda.is_available(), "GPU parity tests need a CUDA device"
    return torch.device("cuda", 0)


def run(stack, s, interp, formula="canvas", reduce="max", **kw):
    raw = torch.from_numpy(np.ascontiguousarray(stack)).to(dev())
    res = deskew_device(raw, s, interp, formula=formula, reduce=reduce, **kw)
    torch.cuda.synchronize()
    vol = None if res.volume is None else res.volume.cpu().numpy()
    return vol, {a: t.cpu().numpy() for a, t in res.projections.items()}


def frame(arr, i, **kw):
    return pl.RawFrame(np.asarray(arr, dtype=np.uint16), i, **kw)


# ---------------------------------------------------------------------------
# golden fixtures produced by the reference itself


@pytest.fixture(params=["tma", "tiled"])
def kernel_path(request, monkeypatch):
    """Run a test through the TMA persistent kernel and through the tiled fallback."""
    if request.param == "tiled":
        monkeypatch.setenv("SSB_DISABLE_TMA", "1")
    else:
        monkeypatch.delenv("SSB_DISABLE_TMA", raising=False)
    return request.param


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
@pytest.mark.parametrize("reduce", ["max", "sum"])
def test_fused_kernel_matches_reference_fixtures(case, reduce, kernel_path):
    st, s, interp = case["stack"], float(case["shear"]), str(case["interp"])
    for formula, key in (("canvas", "vol"), ("npinterp", "batch_vol")):
        vol, pr = run(st, s, interp, formula, reduce)
        np.testing.assert_array_equal(vol, case[key], err_msg=f"{formula} volume")
        for ax in (0, 1, 2):
            np.testing.assert_array_equal(pr[ax], O.project(case[key], ax, reduce),
                                          err_msg=f"{formula} axis {ax}")


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_dropin_canvas_and_batch_match_fixtures(case):
    st, s, interp = case["stack"], float(case["shear"]), str(case["interp"])
    n, h, w = st.shape
    g = geom(n=n, w=w, h=h)
    c = pl.ProjectionCanvas(g, s, interp=interp)
    for i in range(n):
        assert c.place(frame(st[i], i)) == tuple(case["spans"][i])
    np.testing.assert_array_equal(c.finalize_global(), case["xy"])
    np.testing.assert_array_equal(ph.reference_deskew(list(st), g, s, interp=interp), case["batch_xy"])


def test_rolling_matches_reference_fixture():
    r = dict(np.load(f"{GOLDEN}/rolling.npz"))
    for k in range(int(r["count"])):
        n, h, w = (int(v) for v in r[f"c{k}_meta"])
        s, interp = float(r[f"c{k}_shear"]), str(r[f"c{k}_interp"])
        c = pl.ProjectionCanvas(geom(n=n, w=w, h=h), s, interp=interp, mode="rolling")
        for step, (i, px) in enumerate(zip(r[f"c{k}_slices"], r[f"c{k}_frames"])):
            c.rolling_replace(pl.RawFrame(px, int(i)))
            np.testing.assert_array_equal(c.max_pixels, r[f"c{k}_step{step}_max"])
            np.testing.assert_array_equal(c.contributor, r[f"c{k}_step{step}_contrib"])
        c.replace_all(float(r[f"c{k}_shear2"]))
        np.testing.assert_array_equal(c.max_pixels, r[f"c{k}_after_replace_max"])
        np.testing.assert_array_equal(c.contributor, r[f"c{k}_after_replace_contrib"])


def test_warp_matches_reference_fixture():
    wz = dict(np.load(f"{GOLDEN}/warp.npz"))
    k = 0
    while f"in_{k}" in wz:
        out = pl.warp_projection(wz[f"in_{k}"], float(wz[f"scale_{k}"]))
        np.testing.assert_array_equal(out, wz[f"out_{k}"])
        k += 1


# ---------------------------------------------------------------------------
# the reference suite's hand examples, through the drop-in API
# (pkg/tests/test_pipeline.py:107-304, pkg/tests/test_phantom.py:233-272)


class TestPlacementNearest:
    def test_two_slice_hand_example(self):
        c = pl.ProjectionCanvas(geom(n=2), shear_px=1.0, interp="nearest")
        assert (c.width, c.height) == (2, 3)
        c.place(frame([[1, 2], [3, 4]], 0))
        c.place(frame([[5, 0], [0, 1]], 1))
        np.testing.assert_array_equal(c.finalize_global(), [[1, 2], [5, 4], [0, 1]])

    def test_three_slice_hand_example(self):
        c = pl.ProjectionCanvas(geom(n=3), shear_px=1.0, interp="nearest")
        assert c.height == 4
        for i, a in enumerate(([[1, 2], [3, 4]], [[5, 0], [0, 1]], [[2, 9], [6, 3]])):
            c.place(frame(a, i))
        np.testing.assert_array_equal(c.finalize_global(), [[1, 2], [5, 4], [2, 9], [6, 3]])

    def test_order_independent(self):
        rng = np.random.default_rng(7)
        frames = [frame(rng.integers(0, 4096, size=(4, 6)), i) for i in range(5)]
        g = geom(n=5, w=6, h=4)
        c1 = pl.ProjectionCanvas(g, 1.6, interp="nearest")
        c2 = pl.ProjectionCanvas(g, 1.6, interp="nearest")
        for f in frames:
            c1.place(f)
        for f in reversed(frames):
            c2.place(f)
        np.testing.assert_array_equal(c1.finalize_global(), c2.finalize_global())

    def test_fractional_shear_rounds_offset(self):
        assert pl.ProjectionCanvas(geom(n=2), shear_px=0.5, interp="nearest").row_span(1) == (1, 2)

    def test_deskew_place_alias(self):
        c = pl.ProjectionCanvas(geom(n=2), shear_px=1.0, interp="nearest")
        assert pl.deskew_place(c, frame([[1, 2], [3, 4]], 0)) == (0, 1)


class TestPlacementLinear:
    def test_integer_shear_matches_nearest(self):
        rng = np.random.default_rng(3)
        frames = [frame(rng.integers(0, 65535, size=(4, 3)), i) for i in range(4)]
        g = geom(n=4, w=3, h=4)
        cn = pl.ProjectionCanvas(g, 2.0, interp="nearest")
        cl = pl.ProjectionCanvas(g, 2.0, interp="linear")
        for f in frames:
            cn.place(f)
            cl.place(f)
        np.testing.assert_array_equal(cn.finalize_global(), cl.finalize_global())

    def test_half_pixel_lerp_hand_example(self):
        c = pl.ProjectionCanvas(geom(n=2), shear_px=0.5, interp="linear")
        assert c.row_span(1) == (1, 1)
        assert c.place(frame([[10, 20], [30, 40]], 1)) == (1, 1)
        np.testing.assert_array_equal(c.max_pixels[1], [20, 30])

    def test_rounding_to_uint16(self):
        c = pl.ProjectionCanvas(geom(n=2), shear_px=0.5, interp="linear")
        c.place(frame([[0, 1], [1, 2]], 1))
        np.testing.assert_array_equal(c.max_pixels[1], [0, 2])


class TestCanvasValidation:
    def test_wrong_width(self):
        with pytest.raises(ParameterError, match="width"):
            pl.ProjectionCanvas(geom(n=2), 1.0).place(frame(np.zeros((2, 3)), 0))

    def test_wrong_height(self):
        with pytest.raises(ParameterError, match="height"):
            pl.ProjectionCanvas(geom(n=2), 1.0).place(frame(np.zeros((3, 2)), 0))

    def test_slice_out_of_range(self):
        with pytest.raises(ParameterError, match="out of range"):
            pl.ProjectionCanvas(geom(n=2), 1.0).place(frame(np.zeros((2, 2)), 2))

    def test_span_outside_canvas(self):
        c = pl.ProjectionCanvas(geom(n=2), 1.0)
        c.shear_px = 50.0
        with pytest.raises(CapacityError):
            c.place(frame(np.zeros((2, 2)), 1))

    def test_finalize_before_complete(self):
        c = pl.ProjectionCanvas(geom(n=2), 1.0)
        c.place(frame(np.zeros((2, 2)), 0))
        with pytest.raises(ProtocolError, match="1 slice"):
            c.finalize_global()

    def test_finalize_resets(self):
        c = pl.ProjectionCanvas(geom(n=2), 1.0)
        c.place(frame([[1, 2], [3, 4]], 0))
        c.place(frame([[5, 0], [0, 1]], 1))
        c.finalize_global()
        assert c.placed_count == 0
        assert c.max_pixels.max() == 0


class TestRollingMode:
    def test_full_ring_matches_global(self):
        rng = np.random.default_rng(11)
        frames = [frame(rng.integers(0, 65535, size=(4, 3)), i) for i in range(5)]
        g = geom(n=5, w=3, h=4)
        cg = pl.ProjectionCanvas(g, 1.3, interp="linear", mode="global")
        cr = pl.ProjectionCanvas(g, 1.3, interp="linear", mode="rolling")
        for f in frames:
            cg.place(f)
            cr.rolling_replace(f)
        np.testing.assert_array_equal(cr.max_pixels, cg.finalize_global())

    def test_replace_hand_example(self):
        c = pl.ProjectionCanvas(geom(n=2), 1.0, interp="nearest", mode="rolling")
        c.rolling_replace(frame([[1, 2], [3, 4]], 0))
        c.rolling_replace(frame([[5, 0], [0, 1]], 1))
        np.testing.assert_array_equal(c.max_pixels, [[1, 2], [5, 4], [0, 1]])
        c.rolling_replace(frame([[9, 0], [0, 0]], 0, sweep_index=1))
        np.testing.assert_array_equal(c.max_pixels, [[9, 0], [5, 0], [0, 1]])

    def test_contributor_map(self):
        c = pl.ProjectionCanvas(geom(n=2), 1.0, interp="nearest", mode="rolling")
        c.rolling_replace(frame([[1, 2], [3, 4]], 0))
        c.rolling_replace(frame([[5, 0], [0, 1]], 1))
        assert c.contributor[1, 0] == 1
        assert c.contributor[1, 1] == 0
        assert set(np.unique(c.contributor)) <= {-1, 0, 1}

    def test_replace_on_global_rejected(self):
        with pytest.raises(ProtocolError):
            pl.ProjectionCanvas(geom(n=2), 1.0, mode="global").rolling_replace(frame(np.zeros((2, 2)), 0))

    def test_replace_all_new_shear_matches_fresh(self):
        rng = np.random.default_rng(5)
        frames = [frame(rng.integers(0, 65535, size=(3, 4)), i) for i in range(4)]
        g = geom(n=4, w=4, h=3)
        c = pl.ProjectionCanvas(g, 0.8, interp="linear", mode="rolling")
        for f in frames:
            c.rolling_replace(f)
        c.replace_all(1.7)
        fresh = pl.ProjectionCanvas(g, 1.7, interp="linear", mode="rolling")
        for f in frames:
            fresh.rolling_replace(f)
        assert c.max_pixels.shape == fresh.max_pixels.shape
        np.testing.assert_array_equal(c.max_pixels, fresh.max_pixels)

    def test_rolling_window_matches_global_after_sweeps(self):  # test_acceptance.py:121-142
        rng = np.random.default_rng(11)
        g = geom(n=8, w=10, h=12, alpha=60.0, step=0.2, pitch=0.1)
        pixels = rng.integers(0, 65536, (8, 12, 10)).astype(np.uint16)
        from paper_2211_00645_b200.geometry import native_shear_px
        for interp in ("nearest", "linear"):
            for s in (0.0, native_shear_px(g), 1.37):
                whole = pl.ProjectionCanvas(g, s, interp=interp)
                for i in range(8):
                    whole.place(pl.RawFrame(pixels[i], i))
                want = whole.finalize_global()
                roll = pl.ProjectionCanvas(g, s, interp=interp, mode="rolling")
                for sweep in range(3):
                    for i in range(8):
                        roll.rolling_replace(pl.RawFrame(pixels[i], i, sweep_index=sweep))
                    np.testing.assert_array_equal(roll.max_pixels, want)


class TestWarp:
    def test_identity_is_copy(self):
        proj = np.arange(12, dtype=np.uint16).reshape(4, 3)
        out = pl.warp_projection(proj, 1.0)
        np.testing.assert_array_equal(out, proj)
        assert out is not proj

    def test_upscale_by_two(self):
        np.testing.assert_array_equal(pl.warp_projection(np.array([[0], [10]], np.uint16), 2.0),
                                      [[0], [5], [10], [10]])

    def test_downscale_by_half(self):
        np.testing.assert_array_equal(
            pl.warp_projection(np.array([[0], [10], [20], [30]], np.uint16), 0.5), [[0], [20]])


class TestReferenceDeskew:
    def test_single_frame_unchanged(self):
        f = np.arange(12, dtype=np.uint16).reshape(4, 3)
        np.testing.assert_array_equal(ph.reference_deskew([f], geom(n=1, h=4, w=3), 1.5), f)

    def test_two_frames_abut(self):
        f0 = np.array([[1, 2], [3, 4]], np.uint16)
        f1 = np.array([[5, 6], [7, 8]], np.uint16)
        np.testing.assert_array_equal(ph.reference_deskew([f0, f1], geom(n=2), 2.0), np.vstack([f0, f1]))

    def test_accepts_rawframes(self):
        frames = [pl.RawFrame(np.full((2, 2), 5, np.uint16), 0), pl.RawFrame(np.full((2, 2), 9, np.uint16), 1)]
        np.testing.assert_array_equal(ph.reference_deskew(frames, geom(n=2), 0.0), np.full((2, 2), 9))

    def test_streaming_matches_batch_nearest_random(self):  # test_acceptance.py:95-118
        rng = np.random.default_rng(7)
        from paper_2211_00645_b200 import geometry as G
        for _ in range(50):
            n, h, w = int(rng.integers(1, 17)), int(rng.integers(2, 33)), int(rng.integers(2, 33))
            g = G.SheetGeometry(alpha_deg=float(rng.uniform(10.0, 80.0)),
                                scan_step_um=float(rng.uniform(0.05, 0.5)),
                                pixel_pitch_um=float(rng.uniform(0.05, 0.3)),
                                slice_count=n, frame_width_px=w, frame_height_px=h)
            s = float(rng.uniform(0.0, G.max_shear_px(g)))
            frames = [pl.RawFrame(rng.integers(0, 65536, (h, w)).astype(np.uint16), i) for i in range(n)]
            c = pl.ProjectionCanvas(g, s, interp="nearest")
            for f in frames:
                c.place(f)
            np.testing.assert_array_equal(c.finalize_global(), ph.reference_deskew(frames, g, s, "nearest"))


# ---------------------------------------------------------------------------
# randomized + edge cases vs the C oracle


@pytest.mark.parametrize("seed", range(12))
def test_random_shapes_vs_oracle(seed, kernel_path):
    rng = np.random.default_rng(1000 + seed)
    n, h, w = int(rng.integers(1, 40)), int(rng.integers(1, 90)), int(rng.integers(1, 600))
    s = float(rng.choice([rng.uniform(0, 3), 0.8660254037844386, 0.7071067811865476, 1.0, 0.5, 0.0]))
    st = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
    for interp in ("linear", "nearest"):
        for formula in ("canvas", "npinterp"):
            for reduce in ("max", "sum"):
                want_vol, want = C.deskew(st, s, interp, formula, reduce=reduce)
                vol, pr = run(st, s, interp, formula, reduce)
                np.testing.assert_array_equal(vol, want_vol)
                for ax in (0, 1, 2):
                    np.testing.assert_array_equal(pr[ax], want[ax])


def test_unaligned_and_ragged_buffers():
    rng = np.random.default_rng(3)
    st = rng.integers(0, 65536, (9, 33, 136)).astype(np.uint16)
    base = torch.from_numpy(st.reshape(-1)).to(dev())
    buf = torch.empty(base.numel() + 1, dtype=torch.uint16, device=dev())
    buf[1:].copy_(base)
    raw = buf[1:].view(9, 33, 136)  # 2-byte offset: forces the scalar path
    res = deskew_device(raw, 0.83, "linear")
    torch.cuda.synchronize()
    want_vol, want = C.deskew(st, 0.83, "linear")
    np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
    for ax in (0, 1, 2):
        np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])


def test_slab_window_uses_global_indices(kernel_path):
    rng = np.random.default_rng(9)
    st = rng.integers(0, 65536, (60, 50, 264)).astype(np.uint16)
    s = 0.7071067811865476
    full_vol, full = C.deskew(st, s, "linear", reduce="sum")
    U = full_vol.shape[1]
    # slab 20..45 over its own canvas band, as a multi-GPU rank would
    lo = O.linear_span(20, s, 50)[0]
    hi = O.linear_span(44, s, 50)[1]
    vol, pr = run(st[20:45], s, "linear", reduce="sum", first_slice=20, canvas_rows=U,
                  u_begin=lo, u_count=hi - lo + 1)
    np.testing.assert_array_equal(vol, full_vol[20:45, lo:hi + 1])
    np.testing.assert_array_equal(pr[1], full[1][20:45])
    np.testing.assert_array_equal(pr[2], full[2][20:45, lo:hi + 1])


def test_streamer_chunks_match_single_launch(kernel_path):
    from paper_2211_00645_b200.stream import StackStreamer, pinned_stack
    rng = np.random.default_rng(4)
    n, h, w, s = 37, 48, 256, 0.8660254037844386
    st = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
    want_vol, want = C.deskew(st, s, "linear")
    pin = pinned_stack(n, h, w)
    pin[:] = st
    for src in (st, pin):
        for reduce in ("max", "sum"):
            streamer = StackStreamer(h, w, chunk_frames=5, tail_frames=2 if reduce == "max" else None)
            res = streamer.run(src, s, "linear", reduce=reduce)
            torch.cuda.synchronize()
            _, want_r = C.deskew(st, s, "linear", reduce=reduce)
            np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
            for ax in (0, 1, 2):
                np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want_r[ax])


@pytest.mark.parametrize("w", [300, 301, 298])
def test_streamer_odd_width_chunks(w):
    """Chunked streaming (global slice offsets, the uint32 XY accumulator) over rows that are 8-, 2- or
    4-byte aligned: the row-class TMA mode per chunk equals one launch over the whole stack."""
    from paper_2211_00645_b200.stream import StackStreamer, pinned_stack
    rng = np.random.default_rng(w)
    n, h, s = 29, 44, 0.8660254037844386
    st = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
    pin = pinned_stack(n, h, w)
    pin[:] = st
    for interp in ("linear", "nearest"):
        for reduce in ("max", "sum"):
            want_vol, want = C.deskew(st, s, interp, reduce=reduce)
            res = StackStreamer(h, w, chunk_frames=6).run(pin, s, interp, reduce=reduce)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
            for ax in (0, 1, 2):
                np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])


def test_deskew_volume_host_api():
    rng = np.random.default_rng(8)
    st = rng.integers(0, 4096, (12, 20, 40)).astype(np.uint16)
    g = geom(n=12, w=40, h=20)
    res = deskew_volume(st, g, 0.9, "linear", reduce="sum", projection_axes=(0, 2))
    want_vol, want = C.deskew(st, 0.9, "linear", reduce="sum")
    np.testing.assert_array_equal(res.volume, want_vol)
    assert set(res.projections) == {0, 2}
    np.testing.assert_array_equal(res.xy, want[0])
    np.testing.assert_array_equal(res.yz, want[2])


def test_launches_are_counted():
    before = _lib.launch_count()
    run(np.zeros((2, 8, 16), np.uint16), 1.0, "linear")
    assert _lib.launch_count() > before


def test_channel_crops_deskew_in_place(kernel_path):
    """Channel crops (ss/pipeline.py:105-112) passed as strided device views, no copy."""
    from paper_2211_00645_b200.ingest import channel_views

    rng = np.random.default_rng(17)
    st = rng.integers(0, 65536, (19, 40, 272)).astype(np.uint16)
    # channel 0 is unaligned (generic path), channel 1 16-byte aligned (TMA path)
    layout = pl.ChannelLayout(regions=(pl.ChannelRegion(0, 3, 0, 125, 40), pl.ChannelRegion(1, 136, 4, 136, 33)))
    views = channel_views(torch.from_numpy(st).to(dev()), layout)
    for r in layout.regions:
        v = views[r.channel_id]
        assert not v.is_contiguous()
        res = deskew_device(v, 0.8660254037844386, "linear", reduce="max")
        torch.cuda.synchronize()
        crop = np.ascontiguousarray(st[:, r.y0:r.y0 + r.height, r.x0:r.x0 + r.width])
        want_vol, want = C.deskew(crop, 0.8660254037844386, "linear")
        np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
        for ax in (0, 1, 2):
            np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])


def test_pinned_ingest_feeds_streamer():
    import os as _os

    from paper_2211_00645_b200.ingest import load_stack
    from paper_2211_00645_b200.stream import StackStreamer

    stack, geom, _ = load_stack(_os.path.join(GOLDEN, "files", "stack.raw"))
    assert torch.from_numpy(stack).is_pinned()
    res = StackStreamer(geom.frame_height_px, geom.frame_width_px, chunk_frames=4).run(stack, 1.3, "linear")
    torch.cuda.synchronize()
    want_vol, want = C.deskew(np.ascontiguousarray(stack), 1.3, "linear")
    np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
    np.testing.assert_array_equal(res.projections[0].cpu().numpy(), want[0])


@pytest.mark.parametrize("seed", range(6))
def test_rolling_incremental_matches_full_remax_with_ties(seed):
    """Incremental band updates (contributor != replaced slot) vs the reference's full
    band re-max at every step; values in [0, 4) force many ties and zeros."""
    rng = np.random.default_rng(500 + seed)
    n, h, w = int(rng.integers(2, 12)), int(rng.integers(2, 14)), int(rng.integers(1, 40))
    s = float(rng.choice([0.0, 0.5, 1.0, rng.uniform(0, 2.5)]))
    interp = str(rng.choice(["nearest", "linear"]))
    c = pl.ProjectionCanvas(geom(n=n, w=w, h=h), s, interp=interp, mode="rolling")
    U = c.height
    ring = [None] * n
    canvas = np.zeros((U, w), np.uint16)
    contrib = np.full((U, w), -1, np.int16)
    for step in range(4 * n):
        i = int(rng.integers(0, n))
        px = rng.integers(0, 4, size=(h, w)).astype(np.uint16)
        ring[i] = px
        c.rolling_replace(pl.RawFrame(px, i, sweep_index=step // n))
        lo, hi = O.span(i, s, h, interp)
        band, cb = O.rolling_band(ring, s, interp, h, w, lo, hi)
        canvas[lo:hi + 1], contrib[lo:hi + 1] = band, cb
        np.testing.assert_array_equal(c.max_pixels, canvas)
        np.testing.assert_array_equal(c.contributor, contrib)
    # a reset with a non-empty ring forces the full-band path from then on
    c.reset()
    canvas[:] = 0
    contrib[:] = -1
    for step in range(n):
        i = int(rng.integers(0, n))
        px = rng.integers(0, 4, size=(h, w)).astype(np.uint16)
        ring[i] = px
        c.rolling_replace(pl.RawFrame(px, i))
        lo, hi = O.span(i, s, h, interp)
        band, cb = O.rolling_band(ring, s, interp, h, w, lo, hi)
        canvas[lo:hi + 1], contrib[lo:hi + 1] = band, cb
        np.testing.assert_array_equal(c.max_pixels, canvas)
        np.testing.assert_array_equal(c.contributor, contrib)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("tall", ["1", "0"])
def test_projection_only_variants(seed, tall, monkeypatch):
    """Projection-only launches pick other kernel instantiations: 8-row tiles for max,
    XY-only sums without XZ/YZ work.  Every combination against the C oracle."""
    monkeypatch.setenv("SSB_TALL_TILES", tall)
    rng = np.random.default_rng(900 + seed)
    n, h, w = int(rng.integers(1, 60)), int(rng.integers(1, 300)), 8 * int(rng.integers(1, 70))
    s = float(rng.choice([rng.uniform(0, 2.2), 0.7071067811865476, 1.0, 0.5]))
    st = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
    for interp in ("linear", "nearest"):
        for formula in (("canvas", "npinterp") if interp == "linear" else ("canvas",)):
            for reduce in ("max", "sum"):
                for axes in ((0,), (0, 1, 2), (1,), (2,)):
                    _, want = C.deskew(st, s, interp, formula, want_volume=False, axes=axes, reduce=reduce)
                    vol, pr = run(st, s, interp, formula, reduce, write_volume=False, projection_axes=axes)
                    assert vol is None
                    for ax in axes:
                        np.testing.assert_array_equal(pr[ax], want[ax], err_msg=f"{interp} {formula} {reduce} {axes}")


def test_empty_and_degenerate_inputs():
    d = dev()
    empty = torch.empty((0, 16, 32), dtype=torch.uint16, device=d)
    res = deskew_device(empty, 1.0, "linear", canvas_rows=16, projection_axes=(0,))
    torch.cuda.synchronize()
    assert res.projections[0].shape == (16, 32)
    assert int(res.projections[0].to(torch.int32).abs().sum()) == 0
    # zero-width canvas window: nothing to do, no error
    raw = torch.ones((3, 4, 8), dtype=torch.uint16, device=d)
    res = deskew_device(raw, 1.0, "linear", u_begin=2, u_count=0, projection_axes=(0,), write_volume=False)
    torch.cuda.synchronize()
    assert res.projections[0].shape == (0, 8)
    with pytest.raises(ParameterError):
        deskew_device(raw, -0.5, "linear")
    with pytest.raises(ParameterError):
        deskew_device(raw.to(torch.int16), 1.0, "linear")
    with pytest.raises(ParameterError, match="empty"):
        ph.reference_deskew([], geom(), 1.0)


def test_deskew_volume_device_api():
    rng = np.random.default_rng(12)
    st = rng.integers(0, 65536, (10, 24, 64)).astype(np.uint16)
    res = deskew_volume(torch.from_numpy(st).to(dev()), geom(n=10, w=64, h=24), 0.73, "nearest",
                        projection_axes=(1,), reduce="sum")
    assert isinstance(res.volume, torch.Tensor) and res.volume.is_cuda
    want_vol, want = C.deskew(st, 0.73, "nearest", reduce="sum")
    np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
    np.testing.assert_array_equal(res.xz.cpu().numpy(), want[1])


@pytest.mark.parametrize("seed", range(6))
def test_projection_only_long_scans_and_slabs(seed):
    """Projection-only launches walk each u-tile's own slice range (conservative span bounds):
    long scans with small shears, tiny / zero / large shears, and slab windows with global
    slice indices, against the C oracle's full volume."""
    rng = np.random.default_rng(4200 + seed)
    n, h = int(rng.integers(150, 420)), int(rng.integers(20, 90))
    w = 8 * int(rng.integers(1, 40))
    s = [0.05, 1e-7, 0.0, 3.3, 0.7071067811865476, 0.31][seed]
    st = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
    interp = "linear" if seed % 2 == 0 else "nearest"
    for reduce in ("max", "sum"):
        full_vol, _ = C.deskew(st, s, interp, reduce=reduce)
        U = full_vol.shape[1]
        a, b = int(rng.integers(0, n // 3)), int(rng.integers(2 * n // 3, n + 1))
        lo = O.span(a, s, h, interp)[0]
        hi = O.span(b - 1, s, h, interp)[1]
        ref = full_vol[a:b, lo:hi + 1]
        for axes in ((0,), (0, 1, 2)):
            _, pr = run(st[a:b], s, interp, reduce=reduce, first_slice=a, canvas_rows=U, u_begin=lo,
                        u_count=hi - lo + 1, write_volume=False, projection_axes=axes)
            for ax in axes:
                np.testing.assert_array_equal(pr[ax], O.project(ref, ax, reduce), err_msg=f"{reduce} {axes} ax{ax}")
        # whole scan
        _, pr = run(st, s, interp, reduce=reduce, write_volume=False, projection_axes=(0, 1, 2))
        for ax in (0, 1, 2):
            np.testing.assert_array_equal(pr[ax], O.project(full_vol, ax, reduce))


def test_place_from_transient_pinned_frames():
    """place() copies pinned frames asynchronously; the canvas keeps each host buffer alive until
    its copy completed, so callers may drop frames right away; the hold list stays bounded."""
    from paper_2211_00645_b200.stream import pinned_stack

    rng = np.random.default_rng(23)
    n, h, w, s = 24, 64, 256, 0.8660254037844386
    st = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
    c = pl.ProjectionCanvas(geom(n=n, w=w, h=h), s, "linear")
    for i in range(n):
        buf = pinned_stack(1, h, w)[0]
        buf[:] = st[i]
        c.place(pl.RawFrame(buf, i))
        del buf
    np.testing.assert_array_equal(c.finalize_global(), O.canvas_max(st, s, "linear"))
    torch.cuda.synchronize()
    c.place(pl.RawFrame(pinned_stack(1, h, w)[0], 0))
    assert len(c._pending_uploads) <= 2


@pytest.mark.parametrize("w,offset", [(12, 0), (20, 2), (260, 0), (262, 0), (263, 0), (516, 4), (136, 6),
                                      (136, 8), (1000, 0)])
def test_generic_path_vector_widths(w, offset):
    """Widths / base offsets that are not TMA-eligible pick the widest access their alignment
    allows (8-, 4- or 2-byte); every one must stay bit-exact, straddling lanes included."""
    rng = np.random.default_rng(w * 10 + offset)
    n, h = 11, 37
    st = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
    e = offset // 2
    buf = torch.empty(n * h * w + e, dtype=torch.uint16, device=dev())
    buf[e:].copy_(torch.from_numpy(st.reshape(-1)).to(dev()))
    raw = buf[e:].view(n, h, w)
    for interp in ("linear", "nearest"):
        for reduce in ("max", "sum"):
            res = deskew_device(raw, 0.8660254037844386, interp, reduce=reduce)
            torch.cuda.synchronize()
            want_vol, want = C.deskew(st, 0.8660254037844386, interp, reduce=reduce)
            np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
            for ax in (0, 1, 2):
                np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])


@pytest.mark.parametrize("rt", [True, False], ids=["rowclass_tma", "row_copy"])
@pytest.mark.parametrize("seed", range(8))
def test_row_copy_mode_randomized(seed, rt):
    """Rows that are not 16-byte aligned take the persistent kernel's row-class TMA mode (one tensor map
    per row residue class, 248-column tiles) or, with SSB_DISABLE_RT=1, its row-copy
    mode (8-byte cp.async or per-row bulk copies): random widths, strided crops at odd offsets, slab
    windows, both reductions, volume and projection-only, forced narrower access classes -- all
    bit-exact."""
    rng = np.random.default_rng(7700 + seed)
    n, h = int(rng.integers(3, 60)), int(rng.integers(1, 80))
    w = int(rng.integers(1, 700))
    if w % 8 == 0:
        w += int(rng.integers(1, 8))
    pad = int(rng.integers(0, 9))  # crop of a wider frame at an odd column offset
    x0 = int(rng.integers(0, pad + 1))
    s = float(rng.choice([0.8660254037844386, 0.7071067811865476, 0.5, 1.37, 0.05]))
    big = rng.integers(0, 65536, (n, h, w + pad)).astype(np.uint16)
    st = np.ascontiguousarray(big[:, :, x0:x0 + w])
    dev_big = torch.from_numpy(big).to(dev())
    raw = dev_big[:, :, x0:x0 + w]
    force = ["", "4", "2"][seed % 3]
    old = os.environ.get("SSB_FORCE_AC")
    os.environ["SSB_FORCE_AC"] = force
    if not rt:
        os.environ["SSB_DISABLE_RT"] = "1"
    try:
        for interp in ("linear", "nearest"):
            for reduce in ("max", "sum"):
                full_vol, full = C.deskew(st, s, interp, reduce=reduce)
                res = deskew_device(raw, s, interp, reduce=reduce)
                torch.cuda.synchronize()
                np.testing.assert_array_equal(res.volume.cpu().numpy(), full_vol)
                for ax in (0, 1, 2):
                    np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), full[ax])
                # slab window, projection-only
                a, b = n // 4, max(n // 4 + 1, 3 * n // 4)
                lo, hi = O.span(a, s, h, interp)[0], O.span(b - 1, s, h, interp)[1]
                res = deskew_device(raw[a:b], s, interp, reduce=reduce, first_slice=a, canvas_rows=full_vol.shape[1],
                                    u_begin=lo, u_count=hi - lo + 1, write_volume=False)
                torch.cuda.synchronize()
                ref = full_vol[a:b, lo:hi + 1]
                for ax in (0, 1, 2):
                    np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), O.project(ref, ax, reduce))
    finally:
        os.environ.pop("SSB_DISABLE_RT", None)
        if old is None:
            os.environ.pop("SSB_FORCE_AC", None)
        else:
            os.environ["SSB_FORCE_AC"] = old


@pytest.mark.parametrize("w", [2044, 2046, 2047, 1020, 499])
@pytest.mark.parametrize("rt", [True, False], ids=["rowclass_tma", "row_copy"])
def test_odd_width_wide_frames(w, rt):
    """Wide frames whose rows are 8-, 4- or 2-byte aligned: many 248-column tiles (row-class TMA) or
    256-column tiles (row-copy), regular and irregular stages, against the C oracle."""
    rng = np.random.default_rng(w)
    n, h, s = 40, 200, 0.8660254037844386
    st = rng.integers(0, 4096, (n, h, w)).astype(np.uint16)
    raw = torch.from_numpy(st).to(dev())
    if not rt:
        os.environ["SSB_DISABLE_RT"] = "1"
    try:
        for interp, reduce in (("linear", "max"), ("linear", "sum"), ("nearest", "max")):
            want_vol, want = C.deskew(st, s, interp, reduce=reduce)
            res = deskew_device(raw, s, interp, reduce=reduce)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
            for ax in (0, 1, 2):
                np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])
            for axes in ((0,), (0, 1, 2)):
                res = deskew_device(raw, s, interp, reduce=reduce, write_volume=False, projection_axes=axes)
                torch.cuda.synchronize()
                for ax in axes:
                    np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])
    finally:
        os.environ.pop("SSB_DISABLE_RT", None)


def test_deskew_graph_replay_matches_direct_calls():
    """A captured fixed-shape call replays the same kernels: equal to direct calls and to the oracle,
    and it follows in-place updates of the input between replays."""
    from paper_2211_00645_b200.deskew import DeskewGraph

    rng = np.random.default_rng(91)
    st = rng.integers(0, 65536, (20, 48, 256)).astype(np.uint16)
    raw = torch.from_numpy(st).to(dev())
    gr = DeskewGraph(raw, 0.8660254037844386, "linear", reduce="max")
    for k in range(2):
        res = gr.replay()
        torch.cuda.synchronize()
        want_vol, want = C.deskew(st, 0.8660254037844386, "linear")
        np.testing.assert_array_equal(res.volume.cpu().numpy(), want_vol)
        for ax in (0, 1, 2):
            np.testing.assert_array_equal(res.projections[ax].cpu().numpy(), want[ax])
        st = rng.integers(0, 65536, st.shape).astype(np.uint16)
        raw.copy_(torch.from_numpy(st))


def test_canvas_host_writes_reach_device():
    """In-place writes into ProjectionCanvas.max_pixels (a mutable array in the reference,
    ss/pipeline.py:267) are uploaded before the next device operation, not dropped."""
    from paper_2211_00645_b200.geometry import SheetGeometry
    from paper_2211_00645_b200.pipeline import ProjectionCanvas, RawFrame

    g = SheetGeometry(alpha_deg=30.0, scan_step_um=0.115, pixel_pitch_um=0.115, slice_count=3,
                      frame_width_px=8, frame_height_px=4)
    c = ProjectionCanvas(g, 1.0, interp="nearest")
    c.max_pixels[0, :] = 500  # caller write into the host copy
    c.place(RawFrame(pixels=np.full((4, 8), 7, dtype=np.uint16), slice_index=1))
    got = c.max_pixels
    assert (got[0] == 500).all() and (got[1:5] == 7).all()
    np.maximum(c.max_pixels[5:6], 9, out=c.max_pixels[5:6])  # ufunc out= into a view
    for i in (0, 2):
        c.place(RawFrame(pixels=np.zeros((4, 8), dtype=np.uint16), slice_index=i))
    out = c.finalize_global()
    assert (out[0] == 500).all() and (out[5] == 9).all() and (out[1:5] == 7).all()
