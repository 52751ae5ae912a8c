"""Benchmark of the fused deskew + XY/XZ/YZ MIP path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 2]

One step = one pass of the hot path over one synthetic stack resident in HBM:
config 2 = 512 frames x 2048 x 2048 uint16, 30 degree sheet, native shear
(step = pitch = 0.115 um), linear interpolation (the reference default), volume
(N, U, W) uint16 written + XY/XZ/YZ max projections.  Inputs (4.3 GB) and
outputs (5.2 GB) are far larger than the 126 MB L2, so no flush is needed.

With ``--gpus N`` (N > 1) the bench runs config 4, the timelapse batch of 64
distinct stacks sharded round-robin by stack over N ranks (one process per GPU,
NCCL; weak scaling): a step deskews one stack per rank -- its next stack, held
resident in HBM, content ``(base + 37 k) mod 4096`` for global stack k -- and
gathers each stack's XY projection to rank 0 (the display rank) on a side
stream, overlapped with the next stack's kernel.  The step time is the max over
ranks of CUDA-event time.  Launched without torchrun, ``--gpus N`` re-executes
itself under ``torch.distributed.run`` with N local ranks; the driver's own
torchrun launch works the same way.  ``--config 5 --gpus N`` splits one long
scan into scan-axis slabs merged with one NCCL reduce.  ``--dry-run --backend
gloo`` exercises the N-rank launch, rendezvous, display gather and max-over-ranks
timing on CPU (no kernels; value null).

``--impl reference`` times the reference's CPU algorithm (the oracle's numpy
restatement of ProjectionCanvas.place + finalize_global, ss/pipeline.py:229-336,
process-parallel over the host cores) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    1: dict(n=128, h=256, w=512, alpha=30.0, name="config1_128x256x512_30deg"),
    2: dict(n=512, h=2048, w=2048, alpha=30.0, name="config2_512x2048x2048_30deg"),
    3: dict(n=200, h=1024, w=1024, alpha=30.0, name="config3_200x1024x1024_30deg_live_stream"),
    4: dict(n=512, h=2048, w=2048, alpha=30.0, name="config4_timelapse_64x512x2048x2048_30deg_by_stack", stacks=64),
    5: dict(n=8192, h=2048, w=2048, alpha=45.0, name="config5_8192x2048x2048_45deg_slabs_sum"),
}
PITCH = STEP = 0.115


def native_shear(alpha):
    return STEP * math.cos(math.radians(alpha)) / PITCH


def canvas_rows(n, h, s):
    return h + math.ceil((n - 1) * s - 1e-9)


SPEC_HBM_GBS = 8000.0  # B200 HBM3e datasheet bandwidth (SURVEY.md §8(d) asks for both)


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def lookup_traffic(n, h, w, interp, outputs, reduce):
    """ncu DRAM bytes per launch of the dominant kernel for exactly this workload shape and
    output set (profiles/traffic.json, keyed "NxHxW/interp/outputs/reduce"), else None."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            table = json.load(f)
    except (OSError, ValueError):
        return None
    v = table.get(f"{n}x{h}x{w}/{interp}/{outputs}/{reduce}")
    return v.get("bytes") if isinstance(v, dict) else v


def algorithmic_bytes(n, h, w, u, volume=True, axes=(0, 1, 2), reduce="max"):
    e = 2 if reduce == "max" else 4
    proj = {0: u * w, 1: n * w, 2: n * u}
    return 2 * n * h * w + (2 * n * u * w if volume else 0) + e * sum(proj[a] for a in axes)


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k].lower() == "active"})
        loaded = sorted(sm)
        med = loaded[len(loaded) // 2] if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle numpy port) on the host cores


def _cpu_worker(args):
    n_frames, first, h, w, s, u, interp, seed = args
    import numpy as np

    from oracle import deskew_oracle as O

    rng = np.random.default_rng(seed)
    # a few distinct frames cycled (per-frame work does not depend on the values; generating
    # every frame would dominate the wall time and hold GBs of host memory per worker)
    frames = rng.integers(0, 4096, size=(min(n_frames, 4), h, w)).astype(np.uint16)
    canvas = np.zeros((u, w), dtype=np.uint16)
    t0 = time.perf_counter()
    for k in range(n_frames):
        lo, hi, rows = O.slice_rows(frames[k % len(frames)], first + k, s, interp, "canvas")
        np.maximum(canvas[lo:hi + 1], rows, out=canvas[lo:hi + 1])  # ss/pipeline.py:321
    return time.perf_counter() - t0


def cpu_reference_sample(cfg, interp, target_s=12.0, cores=None, pool=None):
    """Process-parallel reference port on a bounded sample; returns (GVox/s, detail)."""
    n, h, w = cfg["n"], cfg["h"], cfg["w"]
    s = native_shear(cfg["alpha"])
    u = canvas_rows(n, h, s)
    cores = cores or len(os.sched_getaffinity(0))
    # calibrate one frame single-threaded
    t1 = _cpu_worker((1, n // 2, h, w, s, u, interp, 0))
    per_worker = max(1, min(n, int(target_s / max(t1, 1e-4))))
    jobs = [(per_worker, (k * per_worker) % max(1, n - per_worker), h, w, s, u, interp, k + 1) for k in range(cores)]
    t0 = time.perf_counter()
    if pool is not None:
        times = pool.map(_cpu_worker, jobs)
    else:
        with mp.get_context("fork").Pool(cores) as p:
            times = p.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    frames = per_worker * cores
    busy = max(times)
    gvox = frames * u * w / busy / 1e9
    sample = (f"{frames} frames of {cfg['name']} ({interp}), {cores} processes x {per_worker} frames, "
              f"ProjectionCanvas.place restated in numpy; {busy:.1f} s compute ({wall:.1f} s wall)")
    return gvox, {"cores": cores, "sample": sample, "frames": frames, "seconds": busy,
                  "ms_per_stack_equiv": busy / frames * n * 1e3}


# ---------------------------------------------------------------------------


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    interp = args.interp
    steps = []
    cores = len(os.sched_getaffinity(0))
    # the whole --steps K --warmup W run is bounded: ~60 s of CPU compute split over the K steps
    per_step = min(args.ref_seconds, max(0.5, 60.0 / max(1, args.steps)))
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(max(args.warmup, args.warmup_ref)):
            cpu_reference_sample(cfg, interp, target_s=min(0.5, per_step), cores=cores, pool=pool)
        for _ in range(args.steps):
            gvox, det = cpu_reference_sample(cfg, interp, target_s=per_step, cores=cores, pool=pool)
            steps.append((gvox, det))
    gv = sorted(x[0] for x in steps)[len(steps) // 2]
    det = steps[-1][1]
    n, h, w = cfg["n"], cfg["h"], cfg["w"]
    u = canvas_rows(n, h, native_shear(cfg["alpha"]))
    line = {
        "impl": "reference", "metric": "deskewed GVoxels/s (fused deskew+MIP)", "value": gv,
        "unit": "GVoxels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        # one step = one full stack's worth of the reference's work, extrapolated from the sample
        "ms_per_step": n * u * w / (gv * 1e9) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u16 in / f64 lerp (numpy) / u16 out", "data": "synthetic uniform [0,4096)",
        "config": {"workload": cfg["name"], "interp": interp, "shear_px": native_shear(cfg["alpha"]),
                   "canvas": [u, w], "outputs": "XY max (ProjectionCanvas: the reference's only output)",
                   "global_batch": 1, "seq_len": n, "stacks_per_s_equiv": gv * 1e9 / (n * u * w),
                   "sample_ms": det["seconds"] * 1e3},
        "cpu_baseline": {"value": gv, "unit": "GVoxels/s", "cores": det["cores"], "kind": "port",
                         "sample": det["sample"]},
        "e2e": {"value": gv, "unit": "GVoxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if n * u * w <= (64 << 20):
        # small stacks (config 1): also the reference's batch oracle as-is (fp64 pile, one
        # np.interp per column, ss/phantom.py:359-402), single process
        line["reference_deskew_as_is"] = reference_deskew_as_is_timing(cfg, interp)
    print(json.dumps(line), flush=True)


def reference_deskew_as_is_timing(cfg, interp, reps=3):
    from oracle import deskew_oracle as O

    n, h, w = cfg["n"], cfg["h"], cfg["w"]
    s = native_shear(cfg["alpha"])
    stack = np.random.default_rng(0).integers(0, 4096, size=(n, h, w)).astype(np.uint16)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.reference_deskew_as_is(stack, s, interp)
        ts.append(time.perf_counter() - t0)
    ms = sorted(ts)[len(ts) // 2] * 1e3
    return {"ms_per_stack": ms, "cores": 1, "interp": interp,
            "what": "oracle.reference_deskew_as_is: (n,U,W) fp64 pile, np.interp per column, max/rint/clip"}


def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2211_00645_b200 import _lib
    from paper_2211_00645_b200.deskew import deskew_device
    from paper_2211_00645_b200.stream import StackStreamer, gpu_numa_cpus, near_gpu, pinned_stack

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, h, w = cfg["n"], cfg["h"], cfg["w"]
    s = native_shear(cfg["alpha"])
    u = canvas_rows(n, h, s)
    interp, reduce = args.interp, "max"
    axes = (0, 1, 2)
    stream = torch.cuda.current_stream(dev)

    # synthetic stacks, generated on device: global stack k = (base + 37 k) mod 4096.
    # Config 2 (N = 1): stack 0, deskewed every step.  Config 4: this rank's shard of the
    # timelapse (round-robin by stack, dist.shard_stacks), every stack distinct and resident in
    # HBM when it fits (64 stacks over 2 ranks = 137 GB per rank), else as many as fit, cycled.
    g = torch.Generator(device=dev).manual_seed(1234)
    base = torch.randint(0, 4096, (n, h, w), generator=g, device=dev, dtype=torch.int16)

    def make_stack(k):
        out = torch.empty_like(base)
        for f0 in range(0, n, 64):  # 64-frame pieces: no stack-sized temporaries
            torch.remainder(base[f0:f0 + 64] + (37 * k) % 4096, 4096, out=out[f0:f0 + 64])
        return out.view(torch.uint16)

    timelapse = "stacks" in cfg
    if timelapse:
        from paper_2211_00645_b200 import dist as D

        mine = D.shard_stacks(cfg["stacks"], rank, world)
        stack_bytes = 2 * n * h * w
        free = torch.cuda.mem_get_info(dev)[0]
        # room for the volume, the projections, the e2e staging and a margin
        fit = max(1, int((free - 2 * n * u * w - stack_bytes - (12 << 30)) // stack_bytes))
        raws = [make_stack(k) for k in mine[:min(len(mine), fit)]]
    else:
        mine = [rank]
        raws = [make_stack(rank)]
    del base
    raw = raws[0]
    vol = torch.empty((n, u, w), dtype=torch.uint16, device=dev)
    projs = {0: torch.empty((u, w), dtype=torch.uint16, device=dev),
             1: torch.empty((n, w), dtype=torch.uint16, device=dev),
             2: torch.empty((n, u), dtype=torch.uint16, device=dev)}
    gather = [torch.empty((u, 2 * w), dtype=torch.uint8, device=dev) for _ in range(world)] if world > 1 and rank == 0 else None
    # N > 1: each stack's XY goes to the display rank (NCCL gather over NVLink).  The gather of
    # step k runs on a side stream while step k+1 deskews into the other XY buffer.
    overlap = world > 1 and not args.no_gather_overlap
    xy_bufs = [projs[0], torch.empty_like(projs[0])] if overlap else [projs[0]]
    comm = torch.cuda.Stream(dev) if overlap else None
    pending = [None, None]
    counter = [0]

    def step():
        b = counter[0] % len(xy_bufs)
        stack = raws[counter[0] % len(raws)]  # this rank's next stack of the timelapse
        counter[0] += 1
        if pending[b] is not None:
            with torch.cuda.stream(stream):
                pending[b].wait()  # the gather that read this buffer has finished
            pending[b] = None
        deskew_device(stack, s, interp, reduce=reduce, volume=vol, projections={0: xy_bufs[b], 1: projs[1], 2: projs[2]},
                      stream=stream)
        if world > 1 and not overlap:
            dist.gather(xy_bufs[b].view(torch.uint8), gather, dst=0)
        elif overlap:
            ready = torch.cuda.Event()
            ready.record(stream)
            with torch.cuda.stream(comm):
                comm.wait_event(ready)
                pending[b] = dist.gather(xy_bufs[b].view(torch.uint8), gather, dst=0, async_op=True)

    def drain():
        for b in range(len(pending)):
            if pending[b] is not None:
                with torch.cuda.stream(stream):
                    pending[b].wait()
                pending[b] = None

    for _ in range(args.warmup):
        step()
    drain()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    t_heat = time.perf_counter()
    while time.perf_counter() - t_heat < args.heat_seconds:  # untimed: lets clocks settle / be sampled
        step()
        drain()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    _lib.profile_enable(True)
    _lib.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # stacks whose inputs + outputs would stay in the 126 MB L2 between steps (config 1) flush
    # it before every step and time the steps one by one; big stacks stream through HBM anyway
    footprint = 2 * n * h * w + 2 * n * u * w
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if footprint < (1 << 30) else None
    if flush is None:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        drain()  # the last gathers are inside the timed region
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
    else:
        # event pairs around each step, the flush between them; no host sync inside the loop,
        # so the host enqueues ahead and no launch latency lands inside a timed window
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
        for a0, a1 in pairs:
            with torch.cuda.stream(stream):
                flush.fill_(1)  # untimed: evict the previous step's data from L2
            a0.record(stream)
            step()
            drain()
            a1.record(stream)
        torch.cuda.synchronize()
        ms = sum(a0.elapsed_time(a1) for a0, a1 in pairs) / args.steps
    l2_note = ("inputs %.2f GB and outputs %.2f GB >> 126 MB L2; no flush" % (2 * n * h * w / 1e9, 2 * n * u * w / 1e9)
               if flush is None else "L2 flushed (512 MB write) before each step; steps timed individually")
    # the timed steps' own launches only (the config-1 extras below are not part of them)
    _lib.profile_enable(False)
    kern_ms, kern_n = _lib.profile_read()
    launches = _lib.launch_count() - launches0
    batch = None
    if flush is not None:
        # small stacks (config 1): the reference's batch oracle (reference_deskew: np.interp rows,
        # pile max, ss/phantom.py:359-402) on the device, XY only, L2 flushed before each call
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
        xy_b = torch.empty((u, w), dtype=torch.uint16, device=dev)
        for a0, a1 in pairs:
            with torch.cuda.stream(stream):
                flush.fill_(1)
            a0.record(stream)
            deskew_device(raw, s, interp, formula="npinterp", projection_axes=(0,), write_volume=False,
                          projections={0: xy_b}, stream=stream)
            a1.record(stream)
        torch.cuda.synchronize()
        bt = sorted(a0.elapsed_time(a1) for a0, a1 in pairs)
        batch = {"ms_per_stack": bt[len(bt) // 2], "what": "phantom.reference_deskew formula (SSB_FORMULA_NPINTERP), "
                 "XY max only, device-resident stack, L2 flushed before each call"}
        if world == 1:
            # the same step replayed from a CUDA graph (deskew.DeskewGraph: scratch reset + fused
            # kernel + finalize as one graph), L2 flushed before each replay
            from paper_2211_00645_b200.deskew import DeskewGraph

            dg = DeskewGraph(raw, s, interp, reduce=reduce)
            for _ in range(3):
                dg.replay()
            for a0, a1 in pairs:
                with torch.cuda.stream(stream):
                    flush.fill_(1)
                a0.record(stream)
                dg.replay()
                a1.record(stream)
            torch.cuda.synchronize()
            gt = sorted(a0.elapsed_time(a1) for a0, a1 in pairs)
            batch["cuda_graph_step_ms"] = gt[len(gt) // 2]
            del dg
    batched = None
    if flush is not None and world == 1 and args.batch > 1:
        batched = run_batched(args, raw, s, interp, reduce, n, h, w, u, dev, stream)
    del flush
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms, kern_ms / max(kern_n, 1)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_avg = float(t[0]), float(t[1])
    else:
        kern_avg = kern_ms / max(kern_n, 1)

    vox = n * u * w
    value = world * vox / (ms * 1e-3) / 1e9
    bytes_launch = algorithmic_bytes(n, h, w, u, True, axes, reduce)
    peak, peak_kind = peaks()
    achieved = bytes_launch / (kern_avg * 1e-3) / 1e9
    traffic = lookup_traffic(n, h, w, interp, "volume+xy,xz,yz", reduce)

    # end-to-end through the public streaming API: pinned host stack -> H2D (2 copy
    # streams) -> fused deskew on device -> projections D2H, every step
    e2e = None
    if not args.no_e2e:
        host = pinned_stack(n, h, w, device=dev)
        host[:] = raw.cpu().numpy()
        streamer = StackStreamer(h, w, device=dev, chunk_frames=args.chunk_frames or None)
        out_host = {a: torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True) for a, t in projs.items()}
        # outputs stay allocated across steps, as in a running acquisition (no per-stack
        # allocation in the loop; the volume stays in HBM)
        from paper_2211_00645_b200.deskew import DeskewResult
        e2e_out = DeskewResult(volume=vol, projections=dict(projs), canvas_rows=u, u_begin=0, u_count=u)

        def e2e_step():
            res = streamer.run(host, s, interp, reduce=reduce, out=e2e_out)
            for a, t in res.projections.items():
                out_host[a].copy_(t, non_blocking=True)
            return res

        for _ in range(max(1, min(2, args.warmup))):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k = max(1, min(args.steps, args.e2e_steps))
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(k):
            res = e2e_step()
            del res
        a1.record(stream)
        torch.cuda.synchronize()
        e_ms = a0.elapsed_time(a1) / k
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        # the bound of this number: a plain pinned 256 MiB H2D copy on this box, measured now
        with near_gpu(dev):
            probe_h = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        probe_d = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        probe_d.copy_(probe_h, non_blocking=True)
        a0.record(stream)
        for _ in range(4):
            probe_d.copy_(probe_h, non_blocking=True)
        a1.record(stream)
        torch.cuda.synchronize()
        ceiling = 4 * (256 << 20) / (a0.elapsed_time(a1) * 1e-3) / 1e9
        del probe_h, probe_d
        h2d = 2 * n * h * w
        e2e = {"value": world * vox / (e_ms * 1e-3) / 1e9, "unit": "GVoxels/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in projs.values()),
               "ms_per_step": e_ms, "h2d_gbs": h2d / (e_ms * 1e-3) / 1e9, "h2d_copy_ceiling_gbs": ceiling, "chunk_frames": streamer.chunk,
               "pinned_on_gpu_numa_node": gpu_numa_cpus(dev) is not None,
               "path": "stream.StackStreamer.run (pinned host -> 2 copy streams -> ssb_deskew per chunk) + projections D2H; volume stays in HBM"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gv, det = cpu_reference_sample(cfg, interp, target_s=args.ref_seconds)
        cpu = {"value": gv, "unit": "GVoxels/s", "cores": det["cores"], "kind": "port", "sample": det["sample"]}

    if rank == 0:
        line = {
            "metric": "deskewed GVoxels/s (fused deskew+MIP)", "value": value, "unit": "GVoxels/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u16 in / fp64-exact lerp (fp32 FFMA2 bracket + fp64 fallback) / u16 out", "data": "synthetic uniform [0,4096), generated on device",
            "config": {"workload": cfg["name"], "interp": interp, "shear_px": s, "canvas": [u, w],
                       "outputs": "volume (N,U,W) u16 + XY/XZ/YZ max", "stacks_per_s": world * 1e3 / ms,
                       "global_batch": world, "seq_len": n, "parallelism": f"dp{world} (stacks)", "l2": l2_note,
                       **({"stacks_total": cfg["stacks"], "stacks_per_rank": len(mine),
                           "resident_distinct_stacks_per_rank": len(raws),
                           "step": "one stack per rank (its next stack of the shard)" +
                                   ("; XY gathered to rank 0 over NCCL on a side stream, overlapped with the next "
                                    "stack" if world > 1 else "")}
                          if timelapse else {})},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "spec_peak": SPEC_HBM_GBS, "frac_of_spec": achieved / SPEC_HBM_GBS,
                         "bytes_per_launch": bytes_launch, "kernel_ms": kern_avg,
                         "kernel": "deskew_tma_kernel (TMA-pipelined persistent)"},
            "clocks": clk, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
        }
        if batch is not None:
            line["reference_deskew_gpu"] = batch
        if batched is not None:
            line["batched"] = batched
        print(json.dumps(line), flush=True)


def run_batched(args, raw, s, interp, reduce, n, h, w, u, dev, stream):
    """Small stacks (config 1): B distinct stacks deskewed by one persistent launch
    (deskew.deskew_batch -> ssb_deskew_batch), volume + 3 MIPs each.  B stacks (1.3 GB at B = 16)
    exceed the L2, so no flush; the main kernel is timed per launch inside libssb."""
    import torch

    from paper_2211_00645_b200 import _lib
    from paper_2211_00645_b200.deskew import deskew_batch

    B = args.batch
    stacks = torch.empty((B, n, h, w), dtype=torch.uint16, device=dev)
    for k in range(B):  # the config-4 rule: stack k = (stack 0 + 37 k) mod 4096
        stacks[k] = ((raw.to(torch.int32) + 37 * k) % 4096).to(torch.uint16)
    res = deskew_batch(stacks, s, interp, reduce=reduce, stream=stream)
    for _ in range(max(3, args.warmup)):
        deskew_batch(stacks, s, interp, reduce=reduce, volume=res.volume, projections=res.projections, stream=stream)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    _lib.profile_read()
    k = max(5, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        deskew_batch(stacks, s, interp, reduce=reduce, volume=res.volume, projections=res.projections, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    kern_ms, kern_n = _lib.profile_read()
    ms = e0.elapsed_time(e1) / k
    kern = kern_ms / max(kern_n, 1)
    nbytes = B * algorithmic_bytes(n, h, w, u, True, (0, 1, 2), reduce)
    peak, peak_kind = peaks()
    return {"stacks_per_launch": B, "ms_per_launch": ms, "value": B * n * u * w / (ms * 1e-3) / 1e9,
            "unit": "GVoxels/s", "stacks_per_s": B * 1e3 / ms, "ms_per_stack": ms / B,
            "roofline": {"bound": "hbm", "achieved": nbytes / (kern * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": nbytes / (kern * 1e-3) / 1e9 / peak, "peak_kind": peak_kind,
                         "bytes_per_launch": nbytes, "kernel_ms": kern,
                         "traffic": lookup_traffic(n, h, w, interp, f"batch{B}/volume+xy,xz,yz", reduce)},
            "what": "deskew.deskew_batch: B distinct stacks (B x 82 MB > L2, no flush), one persistent launch "
                    "(ssb_deskew_batch) + finalize per step"}


def run_stream(args, cfg, rank, world, local_rank):
    """Config 3: continuous live-view stacks through the pinned multi-stream H2D pipeline.

    Every step streams one 200 x 1024 x 1024 stack from pinned host memory (chunks on
    two copy streams, deskew per chunk on the compute stream, XY/XZ/YZ max projections,
    no volume) and copies the projections back.  Throughput = stacks/s over K
    back-to-back stacks; latency = last chunk handed to the copy engine -> projections
    in host memory (the reference's lag_ms, ss/pipeline.py:973), measured per stack.
    """
    import torch

    from paper_2211_00645_b200 import _lib
    from paper_2211_00645_b200.stream import StackStreamer, gpu_numa_cpus, near_gpu, pinned_stack

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, h, w = cfg["n"], cfg["h"], cfg["w"]
    s = native_shear(cfg["alpha"])
    u = canvas_rows(n, h, s)
    host = pinned_stack(n, h, w, device=dev)
    host[:] = np.random.default_rng(rank).integers(0, 4096, size=(n, h, w), dtype=np.uint16)
    streamer = StackStreamer(h, w, device=dev, chunk_frames=args.chunk_frames or None)
    outs = {0: torch.empty((u, w), dtype=torch.uint16, pin_memory=True),
            1: torch.empty((n, w), dtype=torch.uint16, pin_memory=True),
            2: torch.empty((n, u), dtype=torch.uint16, pin_memory=True)}
    cur = torch.cuda.current_stream(dev)

    def step():
        res = streamer.run(host, s, args.interp, reduce="max", write_volume=False)
        for a, t in res.projections.items():
            outs[a].copy_(t, non_blocking=True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(args.steps):
        step()
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = _lib.launch_count() - launches0
    # latency: one stack at a time; event on the copy stream just before the last chunk
    lats = []
    for _ in range(min(args.steps, 10)):
        torch.cuda.synchronize()
        streamer.last_chunk_event = torch.cuda.Event(enable_timing=True)
        step()
        done = torch.cuda.Event(enable_timing=True)
        done.record(cur)
        done.synchronize()
        lats.append(streamer.last_chunk_event.elapsed_time(done))
    lat = sorted(lats)[len(lats) // 2]
    vox = n * u * w
    if rank == 0:
        print(json.dumps({
            "metric": "deskewed GVoxels/s and stacks/s (live-view stream, pinned H2D)", "value": world * vox / (ms * 1e-3) / 1e9,
            "unit": "GVoxels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16 in / fp64-exact lerp (fp32 FFMA2 bracket + fp64 fallback) / u16 out",
            "data": "synthetic uniform [0,4096) in pinned host memory",
            "config": {"workload": cfg["name"], "interp": args.interp, "canvas": [u, w], "stacks_per_s": 1e3 / ms,
                       "latency_ms_last_chunk_to_host": lat, "chunk_frames": streamer.chunk, "tail_frames": streamer.tail,
                       "pinned_on_gpu_numa_node": gpu_numa_cpus(dev) is not None,
                       "outputs": "XY/XZ/YZ max to host every stack, no volume",
                       "h2d_GBps": 2 * n * h * w / (ms * 1e-3) / 1e9},
            "gpu_launches": launches,
        }), flush=True)


def run_slabs(args, cfg, rank, world, local_rank):
    """Config 5: one 8192-frame scan split into contiguous scan-axis slabs (strong scaling).

    Rank r deskews frames [first, first+count) with global slice indices over its canvas
    row window, projection-only, sum XY (uint32); the partial canvases are merged on rank 0
    with one NCCL reduce (uint32 bits as int32 sum) inside the timed step.
    """
    import torch
    import torch.distributed as dist

    from paper_2211_00645_b200 import _lib
    from paper_2211_00645_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, h, w = cfg["n"], cfg["h"], cfg["w"]
    s = native_shear(cfg["alpha"])
    plans = D.plan_slabs(n, h, s, args.interp, world)
    p = plans[rank]
    g = torch.Generator(device=dev).manual_seed(77 + rank)
    raw = torch.empty((p.count, h, w), dtype=torch.uint16, device=dev)
    for k in range(0, p.count, 64):  # generate in chunks (no 2x int32 temporary of the whole slab)
        m = min(64, p.count - k)
        raw[k:k + m] = torch.randint(0, 4096, (m, h, w), generator=g, device=dev, dtype=torch.int32).to(torch.uint16)
    stream = torch.cuda.current_stream(dev)

    def step():
        res = D.deskew_slab(raw, p, s, args.interp, reduce="sum", projection_axes=(0,), stream=stream)
        if world > 1:
            D.combine_xy(res.projections[0], p, w, "sum")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = _lib.launch_count()
    _lib.profile_enable(True)
    _lib.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    kern_ms, kern_n = _lib.profile_read()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    U = p.canvas_rows
    vox = n * U * w
    bytes_launch = 2 * p.count * h * w + 4 * p.u_count * w
    peak, peak_kind = peaks()
    achieved = bytes_launch / (kern_ms / max(kern_n, 1) * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "deskewed GVoxels/s (long scan, scan-axis slabs, sum projection)", "value": vox / (ms * 1e-3) / 1e9,
            "unit": "GVoxels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u16 in / fp64-exact lerp (fp32 FFMA2 bracket + fp64 fallback) / u32 sum",
            "data": "synthetic uniform [0,4096), generated on device",
            "config": {"workload": cfg["name"], "interp": args.interp, "canvas": [U, w],
                       "slab_frames": p.count, "slab_rows": p.u_count, "outputs": "XY sum only (projection-only)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_kind": peak_kind, "bytes_per_launch": bytes_launch,
                         "kernel_ms": kern_ms / max(kern_n, 1),
                         "traffic": lookup_traffic(p.count, h, w, args.interp, "xy", "sum")},
            "gpu_launches": _lib.launch_count() - launches0,
        }), flush=True)


def run_dry(args, cfg, rank, world, local_rank):
    """N-rank plumbing without kernels (CPU test of the multi-GPU launch): rendezvous over the
    chosen backend, per step the display gather of a small uint16 XY tile (dist.gather_to_display,
    the config-4 merge), timing as max over ranks.  Prints the contract line with value null."""
    import torch
    import torch.distributed as dist

    from paper_2211_00645_b200 import dist as D

    xy = torch.full((64, 64), rank + 1, dtype=torch.uint16)
    got = None
    for _ in range(args.warmup):
        got = D.gather_to_display(xy)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        got = D.gather_to_display(xy)
    dist.barrier()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([ms], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ok = got is not None and [int(g[0, 0]) for g in got] == list(range(1, world + 1))
        print(json.dumps({
            "metric": "deskewed GVoxels/s (fused deskew+MIP)", "value": None, "unit": "GVoxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(t[0]), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "none (dry run)", "dry_run": True,
            "config": {"workload": cfg["name"], "backend": args.backend, "parallelism": f"dp{world} (stacks)",
                       "stacks_per_rank": len(D.shard_stacks(cfg.get("stacks", world), rank, world)),
                       "display_gather_ok": ok}}), flush=True)


def self_launch(n: int) -> int:
    """Re-execute this command under torch.distributed.run with n local ranks (one per GPU)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nRanks) stay visible
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=None, choices=sorted(CONFIGS),
                    help="default: 2 at one GPU, 4 (timelapse by stack) at N > 1")
    ap.add_argument("--interp", default="linear", choices=["linear", "nearest"])
    ap.add_argument("--heat-seconds", type=float, default=1.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--warmup-ref", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gather-overlap", action="store_true",
                    help="N > 1: gather each step's XY before the next deskew instead of overlapping")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--chunk-frames", type=int, default=0)
    ap.add_argument("--batch", type=int, default=16, help="config 1: stacks per batched launch (0/1: off)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--dry-run", action="store_true", help="N-rank launch/gather/timing plumbing only (no kernels)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        if not args.dry_run:
            import torch

            if torch.cuda.device_count() < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} but {torch.cuda.device_count()} CUDA devices visible")
        sys.exit(self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = 2 if max(world, args.gpus) == 1 else 4
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world if "WORLD_SIZE" in os.environ else args.gpus)
        return
    if args.dry_run:
        import torch.distributed as dist

        dist.init_process_group(args.backend)
        try:
            run_dry(args, cfg, rank, world, local_rank)
        finally:
            dist.destroy_process_group()
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group(args.backend, device_id=torch.device("cuda", local_rank))
    try:
        runner = {3: run_stream, 5: run_slabs}.get(args.config, run_ours)
        runner(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
