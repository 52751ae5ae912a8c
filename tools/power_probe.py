"""Is the sustained-vs-isolated gap of the headline kernel power/clock related?

Times the config-2 fused launch (volume + 3 max MIPs) per launch with CUDA events in three
regimes: back-to-back for ~3 s, isolated (60 ms idle between launches), and back-to-back
again; nvidia-smi samples SM / memory clocks, power and throttle reasons alongside.
"""
import argparse
import math
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00645_b200.deskew import deskew_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--interp", default="linear")
ap.add_argument("--seconds", type=float, default=3.0)
a = ap.parse_args()

samples = []


def sampler(stop):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.mem,power.draw,"
                          "clocks_event_reasons.sw_power_cap,temperature.gpu", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            samples.append((time.perf_counter(), line.strip()))
    p.terminate()


s = math.cos(math.radians(30.0))
g = torch.Generator(device="cuda").manual_seed(1234)
raw = torch.randint(0, 4096, (512, 2048, 2048), generator=g, device="cuda", dtype=torch.int32).to(torch.uint16)
res = deskew_device(raw, s, a.interp)
torch.cuda.synchronize()


def launch():
    deskew_device(raw, s, a.interp, volume=res.volume, projections=res.projections)


def regime(name, gap_s, seconds):
    t_end = time.perf_counter() + seconds
    evs = []
    t0 = time.perf_counter()
    while time.perf_counter() < t_end:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        evs.append((e0, e1))
        if gap_s:
            torch.cuda.synchronize()
            time.sleep(gap_s)
        elif len(evs) % 64 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ms = sorted(x.elapsed_time(y) for x, y in evs)
    win = [l for (t, l) in samples if t0 <= t <= t1]
    cols = list(zip(*[w.split(", ") for w in win])) if win else []

    def med(k):
        try:
            v = sorted(float(x) for x in cols[k])
            return v[len(v) // 2]
        except Exception:
            return None

    capped = sum(1 for c in (cols[3] if cols else []) if c.strip() == "Active")
    print(f"{name:>14}: n={len(ms):4d} median {ms[len(ms) // 2]:.3f} ms  best {ms[0]:.3f}  worst {ms[-1]:.3f} | "
          f"sm {med(0)} MHz mem {med(1)} MHz power {med(2)} W temp {med(4)} C; power-capped samples "
          f"{capped}/{len(win)}", flush=True)


stop = threading.Event()
th = threading.Thread(target=sampler, args=(stop,), daemon=True)
th.start()
time.sleep(0.5)
regime("back-to-back", 0, a.seconds)
regime("isolated", 0.06, a.seconds)
regime("back-to-back", 0, a.seconds)
regime("isolated", 0.02, a.seconds)
stop.set()
