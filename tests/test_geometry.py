"""Host index math of the drop-in vs tables produced by the reference
(ss/geometry.py) and the reference suite's closed-form checks
(pkg/tests/test_geometry.py, pkg/tests/test_acceptance.py:27-56)."""

import math

import numpy as np
import pytest

from paper_2211_00645_b200 import geometry as G
from paper_2211_00645_b200.errors import CapacityError, ParameterError
from ssb_testutil import GOLDEN, geom


def test_spans_and_extent_bit_exact_vs_reference():
    g = dict(np.load(f"{GOLDEN}/geometry.npz"))
    for a, s in enumerate(g["shears"]):
        s = float(s)
        for b, i in enumerate(g["idx"]):
            assert G.nearest_offset(int(i), s) == g["nearest_off"][a, b]
            for c, h in enumerate(g["hs"]):
                assert G.linear_row_span(int(i), s, int(h)) == tuple(g["linear_span"][a, b, c])
        for c, h in enumerate(g["hs"]):
            for interp in ("nearest", "linear"):
                lo, hi = G.slice_spans(0, int(g["idx"].max()) + 1, s, int(h), interp)
                for b, i in enumerate(g["idx"]):
                    want = (g["nearest_off"][a, b], g["nearest_off"][a, b] + h - 1) if interp == "nearest" \
                        else tuple(g["linear_span"][a, b, c])
                    assert (lo[i], hi[i]) == tuple(want)
        for b, n in enumerate(g["ns"]):
            for c, h in enumerate(g["hs"]):
                gg = geom(n=int(n), h=int(h), w=4)
                assert G.output_extent(gg, s, max_pixels=10**15)[1] == g["extent_height"][a, b, c]


def test_native_shear_closed_forms():
    for alpha in range(5, 90, 5):
        g = G.SheetGeometry(alpha_deg=float(alpha), scan_step_um=0.23, pixel_pitch_um=0.117,
                            slice_count=8, frame_width_px=4, frame_height_px=4)
        s0 = G.native_shear_px(g)
        assert G.view_angle_from_shear(s0, g) == pytest.approx(90.0 - alpha, abs=1e-9)
        assert G.warp_factor(s0, g) == pytest.approx(1.0, abs=1e-9)
    assert G.shear_factor(1.0, 60.0) == pytest.approx(0.5, abs=1e-12)
    assert G.shear_factor(1.0, 45.0) == pytest.approx(math.sqrt(2) / 2, abs=1e-12)


def test_view_transform_roundtrip_and_clamp():
    g = geom(n=8, w=4, h=4, alpha=30.0, step=0.115, pitch=0.115)
    for th in (0.0, 10.0, 45.0, 59.0):
        vt = G.view_transform(g, view_angle_deg=th)
        assert vt.view_angle_deg == pytest.approx(th, abs=1e-9)
    vt = G.view_transform(g, shear_px=1e9)
    assert vt.shear_px == pytest.approx(G.max_shear_px(g))
    with pytest.raises(ParameterError):
        G.view_transform(g)
    with pytest.raises(ParameterError):
        G.view_transform(g, shear_px=1.0, view_angle_deg=3.0)


def test_benchmark_config_extents():
    # canvas U for the five configs
    s30 = G.native_shear_px(G.SheetGeometry(30.0, 0.115, 0.115, 512, 2048, 2048))
    s45 = G.native_shear_px(G.SheetGeometry(45.0, 0.115, 0.115, 8192, 2048, 2048))
    assert G.output_extent(G.SheetGeometry(30.0, 0.115, 0.115, 128, 512, 256), s30) == (512, 366)
    assert G.output_extent(G.SheetGeometry(30.0, 0.115, 0.115, 512, 2048, 2048), s30) == (2048, 2491)
    assert G.output_extent(G.SheetGeometry(30.0, 0.115, 0.115, 200, 1024, 1024), s30) == (1024, 1197)
    assert G.output_extent(G.SheetGeometry(45.0, 0.115, 0.115, 8192, 2048, 2048), s45,
                           max_pixels=10**9) == (2048, 7840)


def test_errors_match_reference():
    with pytest.raises(ParameterError):
        G.SheetGeometry(0.0, 0.1, 0.1, 2, 2, 2)
    with pytest.raises(ParameterError):
        G.SheetGeometry(30.0, 0.1, 0.1, 0, 2, 2)
    with pytest.raises(ParameterError):
        G.output_extent(geom(), -1.0)
    with pytest.raises(CapacityError):
        G.output_extent(geom(n=10_000, w=30_000, h=30_000), 1.0)
    assert issubclass(ParameterError, ValueError)
