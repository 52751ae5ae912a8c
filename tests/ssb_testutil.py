"""Test helpers shared by the suites (fixtures live in conftest.py)."""

import glob
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def golden_cases():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "case_*.npz"))):
        d = np.load(p)
        out.append({k: d[k] for k in d.files} | {"name": os.path.basename(p)})
    return out


def geom(n=2, w=2, h=2, alpha=60.0, step=0.1, pitch=0.1):
    from paper_2211_00645_b200.geometry import SheetGeometry

    return SheetGeometry(alpha_deg=alpha, scan_step_um=step, pixel_pitch_um=pitch, slice_count=n,
                         frame_width_px=w, frame_height_px=h)
