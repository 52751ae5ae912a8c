"""Multi-GPU dispatch (north_star subsystem 4): stacks across ranks, long scans as slabs.

The reference is single-process (no collectives, no
parallelism strategy); this module adds the first multi-GPU layer, one process
per GPU over ``torch.distributed`` (NCCL on B200, gloo in the CPU tests):

* **timelapse batch, sharded by stack** (config 4): stacks are independent, so
  rank r deskews stacks r, r+P, r+2P, ... with no data-path collective; only the
  finished XY projections travel to the display rank (``gather_to_display``).
* **one long scan, sharded into scan-axis slabs** (config 5): output slice i reads
  only frame i (ss/pipeline.py:283-290), so contiguous slabs need zero halo
  planes.  Rank r deskews frames [first, first+count) with their GLOBAL slice
  indices (offset i*s, unlike reference_deskew's list-local index at
  ss/phantom.py:391) over the canvas rows its slices touch, and the partial
  projections are merged on the display rank: XY by an element-wise reduce
  (max or sum) of the row windows, XZ / YZ by concatenation along the slice axis.

NCCL has no uint16 type, so uint16 maxima travel widened to int32.  uint32 sums
travel bit-cast as int32: two's-complement addition is the same bit operation as
uint32 addition, so the int32 SUM is exactly the uint32 sum (mod 2^32, like the
single-GPU kernel's u32 reduction) at half the bytes of an int64 widening.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .geometry import row_span, _ceil_snapped


@dataclass(frozen=True)
class SlabPlan:
    """One rank's share of a long scan.

    The rank owns output slices [first, first + count).  Its INPUT may extend by halo planes
    on either side (clipped at the scan ends): frames [in_first, in_first + in_count).  Both
    reference interpolations read only a slice's own frame (ss/pipeline.py:283-290), so the
    default halo is 0; a cross-frame interpolation would read its neighbours from the halo.
    """

    rank: int
    first: int        # global index of the slab's first frame
    count: int        # frames in the slab
    u_begin: int      # first canvas row the slab touches
    u_count: int      # canvas rows it touches
    canvas_rows: int  # U of the whole scan
    halo_lo: int = 0  # halo planes before `first` in the rank's input
    halo_hi: int = 0  # halo planes after the slab

    @property
    def in_first(self) -> int:
        return self.first - self.halo_lo

    @property
    def in_count(self) -> int:
        return self.halo_lo + self.count + self.halo_hi


def canvas_rows_total(n_total: int, height: int, shear_px: float) -> int:
    return height + _ceil_snapped((n_total - 1) * shear_px)  # ss/geometry.py:141


def plan_slabs(n_total: int, height: int, shear_px: float, interp: str, world: int, halo: int = 0) -> list:
    """Contiguous, near-equal slabs; canvas window = [lo(first), hi(last)] (spans are monotone in i);
    ``halo`` input planes on each side of a slab (clipped at the scan ends)."""
    if halo < 0:
        raise ValueError(f"halo must be >= 0, got {halo}")
    U = canvas_rows_total(n_total, height, shear_px)
    base, extra = divmod(n_total, world)
    plans, first = [], 0
    for r in range(world):
        count = base + (1 if r < extra else 0)
        if count == 0:
            plans.append(SlabPlan(r, first, 0, 0, 0, U))
            continue
        lo, _ = row_span(first, shear_px, height, interp)
        _, hi = row_span(first + count - 1, shear_px, height, interp)
        lo, hi = max(lo, 0), min(hi, U - 1)
        plans.append(SlabPlan(r, first, count, lo, hi - lo + 1, U, min(halo, first),
                              min(halo, n_total - first - count)))
        first += count
    return plans


def shard_stacks(n_stacks: int, rank: int, world: int) -> list:
    """Round-robin stack indices for one rank (config 4)."""
    return list(range(rank, n_stacks, world))


def deskew_slab(raw_slab: torch.Tensor, plan: SlabPlan, shear_px: float, interp: str = "linear", *,
                reduce: str = "sum", projection_axes=(0,), write_volume: bool = False, stream=None):
    """Deskew this rank's frames over its canvas row window (device, one fused launch).

    ``raw_slab`` holds the rank's input frames: the slab itself, or slab + halo planes
    (``plan.in_count`` frames starting at global frame ``plan.in_first``)."""
    from .deskew import deskew_device

    n_in = int(raw_slab.shape[0])
    if n_in == plan.in_count and (plan.halo_lo or plan.halo_hi):
        raw_slab = raw_slab[plan.halo_lo:plan.halo_lo + plan.count]  # the owned slices (a view)
    elif n_in != plan.count:
        raise ValueError(f"slab holds {n_in} frames, plan says {plan.count} (+ halo {plan.halo_lo}/{plan.halo_hi})")
    return deskew_device(raw_slab, shear_px, interp, first_slice=plan.first, canvas_rows=plan.canvas_rows,
                         u_begin=plan.u_begin, u_count=plan.u_count, projection_axes=projection_axes,
                         reduce=reduce, write_volume=write_volume, stream=stream)


def _wide(t: torch.Tensor, reduce: str) -> torch.Tensor:
    """uint16 maxima widened to int32; uint32 sums bit-cast to int32 (same bits)."""
    return t.to(torch.int32) if reduce == "max" else t.contiguous().view(torch.int32)


def _narrow(t: torch.Tensor, reduce: str) -> torch.Tensor:
    return t.to(torch.uint16) if reduce == "max" else t.view(torch.uint32)


def combine_xy(partial: torch.Tensor, plan: SlabPlan, width: int, reduce: str = "sum", dst: int = 0,
               group=None):
    # ``dst`` is a global rank (torch.distributed's convention for reduce / gather with a group)
    """Merge per-slab XY windows into the full (U, W) canvas on rank ``dst``.

    Every rank places its window into a zeroed full canvas and one NCCL reduce
    (MAX or SUM) combines them; rows outside a slab's window contribute 0, which is
    neutral for both reductions.  Returns the canvas on ``dst`` (uint16 for max,
    uint32 for sum), None elsewhere.
    """
    full = torch.zeros((plan.canvas_rows, width), dtype=torch.int32, device=partial.device)
    if plan.count:
        full[plan.u_begin:plan.u_begin + plan.u_count] = _wide(partial, reduce)
    op = dist.ReduceOp.MAX if reduce == "max" else dist.ReduceOp.SUM
    dist.reduce(full, dst=dst, op=op, group=group)
    if dist.get_rank() != dst:
        return None
    return _narrow(full, reduce)


def gather_slices(partial: torch.Tensor, plans: list, rank: int, length: int, reduce: str = "sum",
                  window: bool = False, dst: int = 0, group=None):
    """Concatenate per-slice projections (XZ: (count, W); YZ: (count, u_count)) on ``dst``.

    ``window=True`` marks YZ rows, whose columns are the slab's canvas-row window:
    they are placed at ``u_begin`` inside a full row of ``length`` = U.
    """
    plan = plans[rank]
    rows = max(p.count for p in plans)
    buf = torch.zeros((rows, length), dtype=torch.int32, device=partial.device)
    if plan.count:
        if window:
            buf[:plan.count, plan.u_begin:plan.u_begin + plan.u_count] = _wide(partial, reduce)
        else:
            buf[:plan.count] = _wide(partial, reduce)
    bufs = [torch.empty_like(buf) for _ in plans] if dist.get_rank() == dst else None
    dist.gather(buf, bufs, dst=dst, group=group)
    if bufs is None:
        return None
    out = torch.cat([b[:p.count] for b, p in zip(bufs, plans)])
    return _narrow(out.contiguous(), reduce)


def gather_to_display(projection: torch.Tensor, dst: int = 0, group=None):
    """Send each rank's finished uint16 projection to the display rank (config 4).

    uint16 travels bit-cast as bytes (a pure copy; neither NCCL nor gloo has a
    16-bit integer type).  Returns the list of projections on ``dst``, None elsewhere.
    """
    t = projection.contiguous().view(torch.uint8)
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(t) for _ in range(world)] if dist.get_rank() == dst else None
    dist.gather(t, bufs, dst=dst, group=group)
    return None if bufs is None else [b.view(torch.uint16) for b in bufs]
