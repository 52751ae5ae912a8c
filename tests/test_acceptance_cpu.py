"""Reference acceptance fixtures (tests/golden/acceptance.npz, made by make_acceptance.py from the
reference itself) checked on CPU: the host geometry reproduces the reference's view transforms,
and the oracle reproduces the reference's canvases and warped images on phantom stacks
(pkg/tests/test_acceptance.py:59-92, :145-171)."""

import math
import os

import numpy as np
import pytest

from oracle import deskew_oracle as O
from paper_2211_00645_b200 import geometry as G
from ssb_testutil import GOLDEN

A = dict(np.load(os.path.join(GOLDEN, "acceptance.npz")))


def g_of(key, stack):
    alpha, step, pitch = (float(v) for v in A[key])
    n, h, w = stack.shape
    return G.SheetGeometry(alpha_deg=alpha, scan_step_um=step, pixel_pitch_um=pitch, slice_count=n,
                           frame_width_px=w, frame_height_px=h)


def rms_of_peak(img, oracle):
    img = img.astype(float)
    peak = max(img.max(), float(oracle.max()))
    return math.sqrt(np.mean((img - oracle) ** 2)) / peak


@pytest.mark.parametrize("k", range(4))
def test_sheared_views_oracle_and_geometry(k):
    st = A["a1_stack"]
    g = g_of("a1_geom", st)
    vt = G.view_transform(g, view_angle_deg=float(A["a1_thetas"][k]))
    assert vt.shear_px == float(A[f"a1_{k}_shear"]) and vt.warp_scale == float(A[f"a1_{k}_warp"])
    canvas = O.canvas_max(st, vt.shear_px, "linear")
    np.testing.assert_array_equal(canvas, A[f"a1_{k}_canvas"])
    np.testing.assert_array_equal(O.warp_projection(canvas, vt.warp_scale), A[f"a1_{k}_image"])
    assert rms_of_peak(A[f"a1_{k}_image"], A[f"a1_{k}_oracle"]) < 0.02  # the reference's own bar


@pytest.mark.parametrize("interp", ["linear", "nearest"])
def test_native_restore_oracle_and_geometry(interp):
    st = A["a2_stack"]
    g = g_of("a2_geom", st)
    vt = G.view_transform(g, shear_px=G.native_shear_px(g))
    assert vt.shear_px == float(A["a2_shear"]) and vt.warp_scale == float(A["a2_warp"])
    canvas = O.canvas_max(st, vt.shear_px, interp)
    np.testing.assert_array_equal(canvas, A[f"a2_{interp}_canvas"])
    np.testing.assert_array_equal(O.warp_projection(canvas, vt.warp_scale), A[f"a2_{interp}_image"])
