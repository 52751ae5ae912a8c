"""Acceptance fixtures: phantom stacks rendered and deskewed by the REFERENCE itself.

Run here (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_acceptance.py

Writes ``acceptance.npz`` next to this file.  It pins the two image-content acceptance tests
of the reference (pkg/tests/test_acceptance.py:59-92 and :145-171) to stored data, so the GPU
suite can run them without the reference: the rendered stacks (``phantom.render_stack``), the
reference's warped live-view images for every tested view angle (``ProjectionCanvas.place`` x N
-> ``finalize_global`` -> ``warp_projection``, ss/pipeline.py:316-457) and, for the first test,
the rotate-then-ray-walk oracle projection (``phantom.oracle_project``) the reference compares
against with an RMS < 2 % of peak tolerance.  Scenes and geometries are the reference test's own.
"""

from __future__ import annotations

import os

import numpy as np

from skewstream import geometry as G
from skewstream import phantom as PH
from skewstream import pipeline as PL

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    # pkg/tests/test_acceptance.py:59-92: 45 deg sheet, sphere + off-centre cylinder, 64 slices
    g1 = G.SheetGeometry(alpha_deg=45.0, scan_step_um=0.1, pixel_pitch_um=0.1, slice_count=64,
                         frame_width_px=64, frame_height_px=91)
    sc1 = PH.PhantomScene(
        primitives=(PH.sphere((3.15, 4.2, 2.2), 1.0, 9000.0, soft_edge_um=0.3),
                    PH.cylinder((3.15, 2.0, 0.8), 0.6, 6000.0, axis=(1, 0, 0), soft_edge_um=0.3)),
        extent_um=(6.3, 6.3, 6.3))
    frames1 = PH.render_stack(sc1, g1)
    stack1 = np.stack([f.pixels for f in frames1]).astype(np.uint16)
    vox = PH.voxelize(sc1, 0.1, extent_um=(6.35, 6.35, 6.35))
    out["a1_stack"] = stack1
    out["a1_geom"] = np.array([g1.alpha_deg, g1.scan_step_um, g1.pixel_pitch_um])
    thetas = (0.0, 30.0, 45.0, 80.0)
    out["a1_thetas"] = np.array(thetas)
    for k, theta in enumerate(thetas):
        vt = G.view_transform(g1, view_angle_deg=theta)
        canvas = PL.ProjectionCanvas(g1, vt.shear_px, interp="linear")
        for f in frames1:
            canvas.place(f)
        proj = canvas.finalize_global()
        img = PL.warp_projection(proj, vt.warp_scale)
        t = np.arange(img.shape[0]) * vt.out_pitch_um
        out[f"a1_{k}_shear"] = np.array(vt.shear_px)
        out[f"a1_{k}_warp"] = np.array(vt.warp_scale)
        out[f"a1_{k}_canvas"] = proj
        out[f"a1_{k}_image"] = img
        out[f"a1_{k}_oracle"] = PH.oracle_project(vox, theta, t_um=t).astype(np.float32)

    # pkg/tests/test_acceptance.py:145-171: native restore makes a sphere isotropic
    g2 = G.SheetGeometry(alpha_deg=60.0, scan_step_um=0.15, pixel_pitch_um=0.1, slice_count=32,
                         frame_width_px=44, frame_height_px=44)
    sc2 = PH.PhantomScene(primitives=(PH.sphere((2.15, 3.2, 1.8), 1.5, 8000.0, soft_edge_um=0.15),),
                          extent_um=(4.3, 5.0, 3.6))
    vt2 = G.view_transform(g2, shear_px=G.native_shear_px(g2))
    frames2 = PH.render_stack(sc2, g2)
    out["a2_stack"] = np.stack([f.pixels for f in frames2]).astype(np.uint16)
    out["a2_geom"] = np.array([g2.alpha_deg, g2.scan_step_um, g2.pixel_pitch_um])
    out["a2_shear"] = np.array(vt2.shear_px)
    out["a2_warp"] = np.array(vt2.warp_scale)
    out["a2_out_pitch"] = np.array(vt2.out_pitch_um)
    for interp in ("linear", "nearest"):
        canvas = PL.ProjectionCanvas(g2, vt2.shear_px, interp=interp)
        for f in frames2:
            canvas.place(f)
        proj = canvas.finalize_global()
        out[f"a2_{interp}_canvas"] = proj
        out[f"a2_{interp}_image"] = PL.warp_projection(proj, vt2.warp_scale)
    path = os.path.join(HERE, "acceptance.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
