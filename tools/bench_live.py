"""SURVEY.md 8(f) rows measured on the GPU: the live channel driver, stack ingest into pinned
memory, and the gray8 display encode.  One JSON line per measurement.

* live driver (`live.ChannelDeskewer.process`, ss/pipeline.py:900-980) on config-3 frames
  (200 x 1024 x 1024, 30 deg) from pinned memory: frames/s in global mode (one emission per
  sweep) and rolling mode (one emission per frame), with the emitted image copied to the host.
* ingest (`ingest.load_stack`, ss/source.py:377-474): a config-3 raw stack + sidecar written to
  /tmp, read back into page-locked memory (page cache warm), GB/s.
* display encode (`display.encode_gray8_device`): device time per call on a config-2 canvas
  (2491 x 2048), events on the stream around the call, against 3 bytes/pixel of traffic.
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_00645_b200 import display, ingest  # noqa: E402
from paper_2211_00645_b200.geometry import SheetGeometry, native_shear_px, view_transform  # noqa: E402
from paper_2211_00645_b200.live import ChannelDeskewer  # noqa: E402
from paper_2211_00645_b200.pipeline import RawFrame  # noqa: E402
from paper_2211_00645_b200.stream import pinned_stack  # noqa: E402

n, h, w = 200, 1024, 1024
g = SheetGeometry(30.0, 0.115, 0.115, n, w, h)
vt = view_transform(g, shear_px=native_shear_px(g))
frames = pinned_stack(n, h, w)
frames[:] = np.random.default_rng(0).integers(0, 4096, size=(n, h, w), dtype=np.uint16)

# ---- live driver
for mode in ("global", "rolling"):
    ch = ChannelDeskewer(0, g, vt, "linear", mode)
    sweeps = 3
    for i in range(n):  # warm-up sweep
        ch.process(RawFrame(frames[i], i, 0, 0, timestamp_ns=i))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    emitted = 0
    for sw in range(1, sweeps + 1):
        for i in range(n):
            im = ch.process(RawFrame(frames[i], i, sw, 0, timestamp_ns=(sw * n + i) * 1000))
            emitted += im is not None
    dt = time.perf_counter() - t0
    print(json.dumps({"what": "live.ChannelDeskewer.process", "mode": mode, "frames": n * sweeps,
                      "frame": [h, w], "frames_per_s": n * sweeps / dt, "ms_per_frame": dt / (n * sweeps) * 1e3,
                      "emissions": emitted, "last_timings": im.timings.as_dict() if im is not None else None}),
          flush=True)

# ---- ingest
with tempfile.TemporaryDirectory() as d:
    raw = os.path.join(d, "stack.raw")
    frames.tofile(raw)
    with open(os.path.join(d, "stack.json"), "w") as f:
        json.dump({"geometry": {"alpha_deg": 30.0, "scan_step_um": 0.115, "pixel_pitch_um": 0.115,
                                "slice_count": n, "frame_width_px": w, "frame_height_px": h},
                   "timing": {"exposure_ms": 1.0, "readout_ms": 1.0}, "frames": n}, f)
    ingest.load_stack(raw)  # page cache warm-up
    for label, reuse in (("fresh pinned buffer per call", False), ("into a reused pinned buffer", True)):
        buf = pinned_stack(n, h, w) if reuse else None
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            stack, _, _ = ingest.load_stack(raw, out=buf)
            best = min(best, time.perf_counter() - t0)
            assert stack.shape == (n, h, w)
        print(json.dumps({"what": f"ingest.load_stack (raw, page cache warm, {label})", "bytes": frames.nbytes,
                          "ms": best * 1e3, "gb_per_s": frames.nbytes / best / 1e9}), flush=True)
    t0 = time.perf_counter()
    plain = np.fromfile(raw, dtype=np.uint16)
    t_np = time.perf_counter() - t0
    print(json.dumps({"what": "np.fromfile of the same file (pageable, single thread; the box's file read rate)",
                      "gb_per_s": plain.nbytes / t_np / 1e9}), flush=True)

# ---- display encode
img = torch.randint(0, 65536, (2491, 2048), dtype=torch.int32, device="cuda").to(torch.uint16)
st = torch.cuda.current_stream()
for _ in range(5):
    display.encode_gray8_device(img)
torch.cuda.synchronize()
times = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    display.encode_gray8_device(img)
    e1.record(st)
    e1.synchronize()
    times.append(e0.elapsed_time(e1))
ms = sorted(times)[len(times) // 2]
print(json.dumps({"what": "display.encode_gray8_device (one cooperative launch)", "image": [2491, 2048],
                  "device_ms_median": ms, "algorithmic_gb_per_s": img.numel() * 3 / (ms * 1e-3) / 1e9}), flush=True)
