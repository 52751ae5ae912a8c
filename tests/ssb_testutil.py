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


def display_cases():
    """(DisplayImage, telemetry, {"gray16": bytes, "gray8": bytes}) from display.npz
    (packets made by the reference's encode_frame_packet, ss/server.py:72-117)."""
    from paper_2211_00645_b200.pipeline import DisplayImage, StageTimings

    d = dict(np.load(os.path.join(GOLDEN, "display.npz")))
    out = []
    for k in range(int(d["count"])):
        t = d[f"timings_{k}"]
        tl = d[f"tele_{k}"]
        ch, sweep, sl = (int(v) for v in d[f"meta_{k}"])
        img = DisplayImage(pixels=d[f"px_{k}"], channel_id=ch, sweep_index=sweep, slice_index=sl,
                           view_angle_deg=float(d[f"angle_{k}"]), mode="rolling" if k % 2 else "global",
                           out_pitch_um=float(d[f"pitch_{k}"]), lateral_pitch_um=0.1,
                           timings=StageTimings(*(float(v) for v in t)) if t.size else None)
        tele = {"fps": float(tl[0]), "drops": {"client": int(tl[1]), "server": int(tl[2])}} if tl.size else None
        out.append((img, tele, {f: d[f"{f}_{k}"].tobytes() for f in ("gray16", "gray8")}))
    return out
