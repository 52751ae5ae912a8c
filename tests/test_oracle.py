"""The CPU oracle is pinned against fixtures produced by the reference itself
(tests/golden/make_golden.py) and against the reference tests' hand examples."""

import numpy as np
import pytest

from oracle import c_oracle as C
from oracle import deskew_oracle as O
from ssb_testutil import GOLDEN, golden_cases

CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_numpy_oracle_matches_reference_rows(case):
    st, s, interp = case["stack"], float(case["shear"]), str(case["interp"])
    # streaming rows: ProjectionCanvas._slice_rows (ss/pipeline.py:283-290)
    vol = O.deskew_volume(st, s, interp, "canvas")
    np.testing.assert_array_equal(vol, case["vol"])
    np.testing.assert_array_equal(vol.max(0), case["xy"])
    np.testing.assert_array_equal(O.canvas_max(st, s, interp), case["xy"])
    # batch rows: reference_deskew (np.interp per column, ss/phantom.py:396-402)
    bvol = O.deskew_volume(st, s, interp, "npinterp")
    np.testing.assert_array_equal(bvol, case["batch_vol"])
    np.testing.assert_array_equal(O.reference_deskew(st, s, interp), case["batch_xy"])
    # the as-is port (pile + np.interp per column) the CPU arm times at config 1
    np.testing.assert_array_equal(O.reference_deskew_as_is(st, s, interp), case["batch_xy"])
    np.testing.assert_array_equal(bvol.max(0), case["batch_xy"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
@pytest.mark.parametrize("reduce", ["max", "sum"])
def test_c_oracle_matches_numpy_oracle(case, reduce):
    st, s, interp = case["stack"], float(case["shear"]), str(case["interp"])
    for formula, key in (("canvas", "vol"), ("npinterp", "batch_vol")):
        vol, pr = C.deskew(st, s, interp, formula, reduce=reduce)
        np.testing.assert_array_equal(vol, case[key])
        for ax in (0, 1, 2):
            np.testing.assert_array_equal(pr[ax], O.project(case[key], ax, reduce))


def test_spans_match_reference_tables():
    g = dict(np.load(f"{GOLDEN}/geometry.npz"))
    for a, s in enumerate(g["shears"]):
        for b, i in enumerate(g["idx"]):
            assert O.nearest_offset(int(i), float(s)) == g["nearest_off"][a, b]
            for c, h in enumerate(g["hs"]):
                assert O.linear_span(int(i), float(s), int(h)) == tuple(g["linear_span"][a, b, c])
        for b, n in enumerate(g["ns"]):
            for c, h in enumerate(g["hs"]):
                assert O.canvas_height(int(n), int(h), float(s)) == g["extent_height"][a, b, c]


def test_warp_matches_reference():
    w = dict(np.load(f"{GOLDEN}/warp.npz"))
    k = 0
    while f"in_{k}" in w:
        np.testing.assert_array_equal(O.warp_projection(w[f"in_{k}"], float(w[f"scale_{k}"])), w[f"out_{k}"])
        np.testing.assert_array_equal(C.warp(w[f"in_{k}"], float(w[f"scale_{k}"])), w[f"out_{k}"])
        k += 1
    assert k >= 5


def test_rolling_band_matches_reference():
    r = dict(np.load(f"{GOLDEN}/rolling.npz"))
    for c in range(int(r["count"])):
        n, h, w = (int(v) for v in r[f"c{c}_meta"])
        s, interp = float(r[f"c{c}_shear"]), str(r[f"c{c}_interp"])
        ring = [None] * n
        U = O.canvas_height(n, h, s)
        canvas = np.zeros((U, w), np.uint16)
        contrib = np.full((U, w), -1, np.int16)
        for step, (i, px) in enumerate(zip(r[f"c{c}_slices"], r[f"c{c}_frames"])):
            ring[int(i)] = px
            lo, hi = O.span(int(i), s, h, interp)
            band, cb = O.rolling_band(ring, s, interp, h, w, lo, hi)
            canvas[lo:hi + 1], contrib[lo:hi + 1] = band, cb
            np.testing.assert_array_equal(canvas, r[f"c{c}_step{step}_max"])
            np.testing.assert_array_equal(contrib, r[f"c{c}_step{step}_contrib"])


# hand examples from the reference suite (pkg/tests/test_pipeline.py:107-179,
# pkg/tests/test_phantom.py:233-254), restated on the oracle

def test_kat_two_slice_nearest():
    st = np.array([[[1, 2], [3, 4]], [[5, 0], [0, 1]]], np.uint16)
    np.testing.assert_array_equal(O.canvas_max(st, 1.0, "nearest"), [[1, 2], [5, 4], [0, 1]])


def test_kat_three_slice_nearest():
    st = np.array([[[1, 2], [3, 4]], [[5, 0], [0, 1]], [[2, 9], [6, 3]]], np.uint16)
    np.testing.assert_array_equal(O.canvas_max(st, 1.0, "nearest"), [[1, 2], [5, 4], [2, 9], [6, 3]])
    np.testing.assert_array_equal(O.reference_deskew(st, 1.0, "nearest"), [[1, 2], [5, 4], [2, 9], [6, 3]])


def test_kat_half_pixel_lerp_and_half_even():
    assert O.linear_span(1, 0.5, 2) == (1, 1)
    lo, hi, rows = O.slice_rows(np.array([[10, 20], [30, 40]], np.uint16), 1, 0.5, "linear")
    np.testing.assert_array_equal(rows, [[20, 30]])
    lo, hi, rows = O.slice_rows(np.array([[0, 1], [1, 2]], np.uint16), 1, 0.5, "linear")
    np.testing.assert_array_equal(rows, [[0, 2]])  # rint half to even


def test_kat_single_frame_and_abutting_frames():
    f = np.arange(12, dtype=np.uint16).reshape(1, 4, 3)
    np.testing.assert_array_equal(O.reference_deskew(f, 1.5), f[0])
    st = np.array([[[1, 2], [3, 4]], [[5, 6], [7, 8]]], np.uint16)
    np.testing.assert_array_equal(O.reference_deskew(st, 2.0), np.vstack([st[0], st[1]]))


def test_slab_restriction_equals_full_volume():
    rng = np.random.default_rng(5)
    st = rng.integers(0, 65536, (20, 30, 17)).astype(np.uint16)
    full, _ = C.deskew(st, 0.77, "linear")
    v, _ = C.deskew(st[5:12], 0.77, "linear", first_slice=5, u_begin=3, u_count=20)
    np.testing.assert_array_equal(v, full[5:12, 3:23])
    np.testing.assert_array_equal(
        O.deskew_volume(st[5:12], 0.77, "linear", first_slice=5, u_begin=3, u_count=20), v)
