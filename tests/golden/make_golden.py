"""Generate golden fixtures by running the REFERENCE implementation itself.

Run here (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It writes small ``.npz`` fixtures next to this file.  Nothing at test time
reads ``/root/reference``; the fixtures travel with the repo.

Sources of truth (reference file:line):
* geometry tables: ``geometry.output_extent`` / ``nearest_offset`` /
  ``linear_row_span`` (ss/geometry.py:129-147, 236-255)
* streaming rows + canvas: ``ProjectionCanvas.row_span`` / ``_slice_rows`` /
  ``place`` / ``finalize_global`` (ss/pipeline.py:274-336) -- the per-slice
  rows give the deskewed volume V[i, lo:hi+1] exactly as the reference
  computes them; the canvas is its axis-0 max
* batch rows: ``phantom.reference_deskew`` (ss/phantom.py:359-402) on one-hot
  stacks (all frames zero but frame i) gives slice i's rounded np.interp rows;
  the full call gives the batch MIP
* warp: ``pipeline.warp_projection`` (ss/pipeline.py:434-457)
* rolling: ``ProjectionCanvas.rolling_replace`` / ``replace_all``
  (ss/pipeline.py:345-398) snapshots of ``max_pixels`` and ``contributor``
* display packets: ``server.encode_frame_packet`` (ss/server.py:72-117), gray16 and gray8
  (``--only display`` regenerates just ``display.npz``)
* live emissions: ``LivePipeline.step`` (ss/pipeline.py:874-980) over scripted frames with
  view / mode changes (``--only live``)
"""

from __future__ import annotations

import os
import sys

import numpy as np

from skewstream import geometry as G
from skewstream import phantom as PH
from skewstream import pipeline as PL

HERE = os.path.dirname(os.path.abspath(__file__))


def geom(n, h, w, alpha=60.0, step=0.2, pitch=0.1):
    return G.SheetGeometry(alpha_deg=alpha, scan_step_um=step, pixel_pitch_um=pitch,
                           slice_count=n, frame_width_px=w, frame_height_px=h)


def canvas_case(stack, s, interp):
    n, h, w = stack.shape
    g = geom(n, h, w)
    c = PL.ProjectionCanvas(g, s, interp=interp)
    vol = np.zeros((n, c.height, w), dtype=np.uint16)
    spans = np.zeros((n, 2), dtype=np.int64)
    for i in range(n):
        f = PL.RawFrame(stack[i], i)
        lo, hi = c.row_span(i)
        spans[i] = (lo, hi)
        vol[i, lo:hi + 1] = c._slice_rows(f, lo, hi)
        c.place(f)
    xy = c.finalize_global()
    return vol, xy, spans


def batch_case(stack, s, interp):
    n, h, w = stack.shape
    g = geom(n, h, w)
    full = PH.reference_deskew(list(stack), g, s, interp=interp)
    vol = np.zeros((n,) + full.shape, dtype=np.uint16)
    for i in range(n):
        onehot = np.zeros_like(stack)
        onehot[i] = stack[i]
        vol[i] = PH.reference_deskew(list(onehot), g, s, interp=interp)
    # the one-hot trick is exact only where slice i is the unique nonzero
    # contributor; restrict the volume golden to slice i's own span
    for i in range(n):
        if interp == "nearest":
            lo = G.nearest_offset(i, s)
            hi = lo + h - 1
        else:
            lo, hi = G.linear_row_span(i, s, h)
        vol[i, :max(lo, 0)] = 0
        vol[i, hi + 1:] = 0
    return vol, full


def main():
    rng = np.random.default_rng(20221101)
    out = {}

    # ---- geometry tables -------------------------------------------------
    shears = np.concatenate([
        rng.uniform(0.0, 3.0, 200),
        np.array([0.0, 0.5, 1.0, 2.0, 1.5, 0.1 * 3, 0.7 + 1e-12, 1.0 - 1e-12,
                  1.0 + 1e-10, 2.0 / 3.0, 1.0 / 3.0, np.cos(np.radians(30.0)),
                  np.cos(np.radians(45.0)), 0.866025403784439, 0.25, 0.125]),
    ])
    idx = np.concatenate([np.arange(0, 160), np.arange(500, 520), np.arange(8180, 8192)])
    hs = np.array([1, 2, 3, 7, 256, 2048])
    tab_lin = np.zeros((shears.size, idx.size, hs.size, 2), dtype=np.int64)
    tab_near = np.zeros((shears.size, idx.size), dtype=np.int64)
    for a, s in enumerate(shears):
        for b, i in enumerate(idx):
            tab_near[a, b] = G.nearest_offset(int(i), float(s))
            for c, h in enumerate(hs):
                tab_lin[a, b, c] = G.linear_row_span(int(i), float(s), int(h))
    ns = np.array([1, 2, 5, 128, 200, 512, 8192])
    ext = np.zeros((shears.size, ns.size, hs.size), dtype=np.int64)
    for a, s in enumerate(shears):
        for b, n in enumerate(ns):
            for c, h in enumerate(hs):
                ext[a, b, c] = G.output_extent(geom(int(n), int(h), 4), float(s),
                                               max_pixels=10**15)[1]
    np.savez_compressed(os.path.join(HERE, "geometry.npz"), shears=shears, idx=idx,
                        hs=hs, ns=ns, linear_span=tab_lin, nearest_off=tab_near,
                        extent_height=ext)

    # ---- volume / canvas / batch cases -----------------------------------
    cases = []
    # (n, h, w, s, interp, hi_value)
    base = [
        (2, 2, 2, 1.0, "nearest", 10),
        (3, 2, 2, 1.0, "nearest", 10),
        (2, 2, 2, 0.5, "linear", 4),
        (2, 2, 2, 0.5, "nearest", 4),
        (4, 4, 3, 2.0, "linear", 65536),
        (5, 4, 6, 1.6, "nearest", 4096),
        (5, 4, 3, 1.3, "linear", 65536),
        (1, 4, 3, 1.5, "linear", 65536),
        (6, 1, 5, 0.7, "linear", 65536),
        (6, 5, 1, 0.7, "linear", 65536),
        (7, 9, 17, 0.0, "linear", 65536),
        (7, 9, 17, 0.0, "nearest", 65536),
        (9, 12, 33, 0.5, "linear", 8),     # exact half ties -> rint half-even
        (9, 12, 33, 0.25, "linear", 65536),
        (16, 32, 40, 1.0 + 1e-10, "linear", 65536),   # offsets within 1e-9 of integers
        (16, 32, 40, 1.0 - 1e-12, "linear", 65536),
        (16, 32, 40, 0.1 * 3, "linear", 65536),
        (16, 32, 40, 2.0 / 3.0, "linear", 65536),
        (16, 32, 40, 2.0 / 3.0, "nearest", 65536),
        (20, 24, 72, float(np.cos(np.radians(30.0))), "linear", 4096),
        (20, 24, 72, float(np.cos(np.radians(30.0))), "nearest", 4096),
        (20, 24, 72, float(np.cos(np.radians(45.0))), "linear", 65536),
        (12, 40, 136, 1.7320508075688772, "linear", 65536),  # 2x native at 30 deg
        (33, 17, 64, 0.3660254037844386, "linear", 65536),
        (24, 40, 264, 0.8660254037844386, "linear", 65536),  # ragged width (not /8)
        (32, 48, 136, 0.8660254037844386, "linear", 4096),
        (32, 48, 136, 0.8660254037844386, "nearest", 4096),
    ]
    for _ in range(14):
        n = int(rng.integers(1, 24))
        h = int(rng.integers(1, 40))
        w = int(rng.integers(1, 70))
        s = float(rng.uniform(0.0, 2.5))
        cases.append((n, h, w, s, str(rng.choice(["nearest", "linear"])), 65536))
    cases = base + cases

    for k, (n, h, w, s, interp, vmax) in enumerate(cases):
        stack = rng.integers(0, vmax, size=(n, h, w)).astype(np.uint16)
        vol, xy, spans = canvas_case(stack, s, interp)
        bvol, bxy = batch_case(stack, s, interp)
        np.savez_compressed(os.path.join(HERE, f"case_{k:03d}.npz"),
                            stack=stack, shear=np.float64(s), interp=interp,
                            vol=vol, xy=xy, spans=spans, batch_vol=bvol, batch_xy=bxy)
        print(f"case {k}: n={n} h={h} w={w} s={s!r} {interp} canvas={xy.shape}", file=sys.stderr)

    # ---- warp ---------------------------------------------------------------
    warp = {}
    for k, (rows, cols, scale) in enumerate([(4, 3, 1.0), (2, 1, 2.0), (4, 1, 0.5),
                                              (37, 11, 1.3), (64, 9, 0.77), (50, 5, 0.9999),
                                              (91, 64, 1.1547005383792517)]):
        proj = rng.integers(0, 65536, size=(rows, cols)).astype(np.uint16)
        warp[f"in_{k}"] = proj
        warp[f"scale_{k}"] = np.float64(scale)
        warp[f"out_{k}"] = PL.warp_projection(proj, scale)
    np.savez_compressed(os.path.join(HERE, "warp.npz"), **warp)

    # ---- rolling ------------------------------------------------------------
    roll = {}
    k = 0
    for (n, h, w, s, interp) in [(5, 4, 3, 1.3, "linear"), (2, 2, 2, 1.0, "nearest"),
                                 (8, 12, 10, 0.5773502691896258, "linear"),
                                 (8, 12, 10, 1.37, "nearest"), (6, 7, 9, 0.0, "linear")]:
        g = geom(n, h, w)
        c = PL.ProjectionCanvas(g, s, interp=interp, mode="rolling")
        frames = []
        # two full sweeps then a partial third, with a shear change in between
        for sweep in range(3):
            order = rng.permutation(n) if sweep == 1 else np.arange(n)
            for i in order[: (n if sweep < 2 else max(1, n // 2))]:
                px = rng.integers(0, 65536, size=(h, w)).astype(np.uint16)
                frames.append((int(i), px))
                c.rolling_replace(PL.RawFrame(px, int(i), sweep_index=sweep))
                roll[f"c{k}_step{len(frames) - 1}_max"] = c.max_pixels.copy()
                roll[f"c{k}_step{len(frames) - 1}_contrib"] = c.contributor.copy()
        c.replace_all(s * 1.5 + 0.1)
        roll[f"c{k}_after_replace_max"] = c.max_pixels.copy()
        roll[f"c{k}_after_replace_contrib"] = c.contributor.copy()
        roll[f"c{k}_meta"] = np.array([n, h, w], dtype=np.int64)
        roll[f"c{k}_shear"] = np.float64(s)
        roll[f"c{k}_shear2"] = np.float64(s * 1.5 + 0.1)
        roll[f"c{k}_interp"] = interp
        roll[f"c{k}_slices"] = np.array([f[0] for f in frames], dtype=np.int64)
        roll[f"c{k}_frames"] = np.stack([f[1] for f in frames])
        k += 1
    roll["count"] = np.int64(k)
    np.savez_compressed(os.path.join(HERE, "rolling.npz"), **roll)

    # ---- recorded-stack files (ss/source.py:377-395) ------------------------
    from skewstream import source as SRC
    fdir = os.path.join(HERE, "files")
    os.makedirs(fdir, exist_ok=True)
    g = geom(6, 10, 24)
    frames = rng.integers(0, 65536, size=(6, 10, 24)).astype(np.uint16)
    SRC.write_stack_raw(os.path.join(fdir, "stack.raw"), list(frames), g)
    SRC.write_stack_tiff(os.path.join(fdir, "stack.tif"), list(frames), g)
    np.save(os.path.join(fdir, "frames.npy"), frames)
    src = SRC.open_stack(os.path.join(fdir, "stack.raw"))
    np.save(os.path.join(fdir, "replayed.npy"), np.stack([src.next_frame().pixels for _ in range(6)]))


def display_cases():
    """display.npz: packets of the reference's encode_frame_packet (own seed)."""
    from skewstream import server as SV
    rng = np.random.default_rng(2211)
    images = [
        np.array([[0, 100], [200, 1000]]), np.full((3, 4), 1234), np.array([[500, 800], [650, 740]]),
        np.array([[7]]), rng.integers(0, 65536, (9, 13)), rng.integers(0, 4096, (64, 48)),
        rng.integers(0, 65536, (60, 257)), 1000 + rng.integers(0, 2, (33, 17)),
        rng.integers(0, 65536, (1, 1001)), np.arange(65536).reshape(256, 256)[:, ::-1],
        rng.integers(30000, 30256, (128, 200)),
    ]
    out = {}
    for k, px in enumerate(images):
        px = np.asarray(px, dtype=np.uint16)
        timings = PL.StageTimings(4.0 + k, 1.5, 0.25, 6.0 + k / 3) if k % 2 else None
        tele = {"fps": 12.5 + k, "drops": {"client": k, "server": 1}} if k % 3 == 1 else None
        img = PL.DisplayImage(pixels=px, channel_id=k % 4, sweep_index=41 + k, slice_index=12 * k,
                              view_angle_deg=30.0 + 1.337 * k, mode="rolling" if k % 2 else "global",
                              out_pitch_um=0.115 + 0.001 * k, lateral_pitch_um=0.1, timings=timings)
        out[f"px_{k}"] = px
        out[f"meta_{k}"] = np.array([k % 4, 41 + k, 12 * k], dtype=np.int64)
        out[f"angle_{k}"] = np.float64(30.0 + 1.337 * k)
        out[f"pitch_{k}"] = np.float64(0.115 + 0.001 * k)
        out[f"timings_{k}"] = (np.array([4.0 + k, 1.5, 0.25, 6.0 + k / 3]) if timings else np.zeros(0))
        out[f"tele_{k}"] = (np.array([12.5 + k, k, 1.0]) if tele else np.zeros(0))
        for fmt in ("gray16", "gray8"):
            out[f"{fmt}_{k}"] = np.frombuffer(SV.encode_frame_packet(img, pixel_format=fmt, telemetry=tele),
                                              dtype=np.uint8).copy()
    out["count"] = np.int64(len(images))
    np.savez_compressed(os.path.join(HERE, "display.npz"), **out)


def live_cases():
    """live.npz: emissions of the reference's LivePipeline (ss/pipeline.py:706-1064) driven
    frame by frame with parameter changes at fixed points (own seed)."""
    from skewstream import geometry as GEO
    from skewstream.clock import VirtualClock
    from skewstream.errors import EndOfStream

    rng = np.random.default_rng(645)

    class Script:
        def __init__(self, g, frames, period_ms):
            self.geom, self.frames, self.k = g, frames, 0
            self.period_ns = int(period_ms * 1e6)
            self.clock = VirtualClock()

        def set_exposure_ms(self, ms):
            pass

        def next_frame(self):
            if self.k >= len(self.frames):
                raise EndOfStream("done")
            sweep, idx, px = self.frames[self.k]
            self.k += 1
            self.clock.sleep_until(self.clock.now_ns() + self.period_ns)
            return PL.RawFrame(pixels=px, slice_index=idx, sweep_index=sweep, channel_id=0,
                               timestamp_ns=self.clock.now_ns())

    scenarios = [
        # (n, h, w, interp, mode, sweeps, changes {frame_count: (kind, value)})
        (6, 10, 12, "linear", "global", 3, {8: ("angle", 35.0)}),
        (5, 7, 9, "nearest", "rolling", 3, {4: ("shear", 1.7), 9: ("mode", "global")}),
        (4, 9, 8, "linear", "global", 4, {3: ("mode", "rolling"), 7: ("angle", 50.0), 11: ("mode", "global")}),
    ]
    out = {}
    for k, (n, h, w, interp, mode, sweeps, changes) in enumerate(scenarios):
        g = geom(n, h, w)
        frames = [(sw, i, rng.integers(0, 65536, (h, w)).astype(np.uint16))
                  for sw in range(sweeps) for i in range(n)]
        if k == 2:  # drop frames mid-sweep: a partial sweep is abandoned
            frames = frames[:5] + frames[6:]
        src = Script(g, frames, 7.0)
        cfg = PL.PipelineConfig(geom=g, mode=mode, interp=interp)
        pipe = PL.LivePipeline(src, cfg)
        vt0 = pipe.vt
        ems, chg = [], []
        for step in range(len(frames)):
            if step in changes:
                kind, val = changes[step]
                if kind == "angle":
                    pipe.post_params(view_angle_deg=val)
                    vt = GEO.view_transform(g, view_angle_deg=val, out_pitch_um=cfg.out_pitch_um)
                elif kind == "shear":
                    pipe.post_params(shear_px=val)
                    vt = GEO.view_transform(g, shear_px=val, out_pitch_um=cfg.out_pitch_um)
                else:
                    pipe.post_params(mode=val)
                    vt = None
                chg.append((step, kind, val, vt))
            for im in pipe.step():
                ems.append((step, im))
        out[f"s{k}_meta"] = np.array([n, h, w, sweeps], dtype=np.int64)
        out[f"s{k}_interp"] = interp
        out[f"s{k}_mode"] = mode
        out[f"s{k}_vt0"] = np.array([vt0.shear_px, vt0.warp_scale, vt0.view_angle_deg, vt0.out_pitch_um])
        out[f"s{k}_frames"] = np.stack([f[2] for f in frames])
        out[f"s{k}_frame_ids"] = np.array([[f[0], f[1]] for f in frames], dtype=np.int64)
        out[f"s{k}_changes"] = np.array([[c[0], ["angle", "shear", "mode"].index(c[1]),
                                          (["global", "rolling"].index(c[2]) if c[1] == "mode" else 0)]
                                         for c in chg], dtype=np.int64)
        out[f"s{k}_change_vt"] = np.array([[c[3].shear_px, c[3].warp_scale, c[3].view_angle_deg, c[3].out_pitch_um]
                                           if c[3] is not None else [0.0] * 4 for c in chg])
        out[f"s{k}_emit_count"] = np.int64(len(ems))
        for e, (step, im) in enumerate(ems):
            out[f"s{k}_e{e}_px"] = im.pixels
            out[f"s{k}_e{e}_ids"] = np.array([step, im.sweep_index, im.slice_index,
                                              ["global", "rolling"].index(im.mode)], dtype=np.int64)
            out[f"s{k}_e{e}_f"] = np.array([im.view_angle_deg, im.out_pitch_um, im.lateral_pitch_um,
                                            im.timings.acquisition_ms])
        print(f"live scenario {k}: {len(frames)} frames, {len(ems)} emissions", file=sys.stderr)
    out["count"] = np.int64(len(scenarios))
    np.savez_compressed(os.path.join(HERE, "live.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--only"]:
        {"display": display_cases, "live": live_cases}[sys.argv[2]]()
    else:
        main()
        display_cases()
        live_cases()
