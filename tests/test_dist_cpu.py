"""Multi-rank logic of dist.py with world_size 2 over gloo on CPU.

The device kernel cannot run here, so each rank computes its slab's partial
projections with the C oracle (the same numbers the kernel produces, see the GPU
parity suite) and the torch.distributed merge paths are exercised for real.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_00645_b200 import dist as D

WORLD = 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, case):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import c_oracle as C

        n, h, w, s, interp, reduce = case
        rng = np.random.default_rng(123)
        stack = rng.integers(0, 65536, (n, h, w)).astype(np.uint16)
        plans = D.plan_slabs(n, h, s, interp, world)
        p = plans[rank]
        _, part = C.deskew(stack[p.first:p.first + p.count], s, interp, first_slice=p.first,
                           u_begin=p.u_begin, u_count=p.u_count, want_volume=False, reduce=reduce)
        xy = D.combine_xy(torch.from_numpy(part[0]), p, w, reduce)
        xz = D.gather_slices(torch.from_numpy(part[1]), plans, rank, w, reduce)
        yz = D.gather_slices(torch.from_numpy(part[2]), plans, rank, p.canvas_rows, reduce, window=True)
        disp = D.gather_to_display(torch.from_numpy(part[0].astype(np.uint16) if reduce == "max"
                                                    else np.zeros((2, 2), np.uint16)))
        if rank == 0:
            np.savez(os.path.join(out_dir, "r0.npz"), xy=xy.numpy(), xz=xz.numpy(), yz=yz.numpy(),
                     disp_n=len(disp))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (37, 20, 24, 0.7071067811865476, "linear", "sum"),
    (37, 20, 24, 0.7071067811865476, "linear", "max"),
    (16, 9, 8, 1.37, "nearest", "max"),
    (5, 12, 16, 0.0, "linear", "sum"),
])
def test_slab_sharding_matches_single_stack(tmp_path, case):
    from oracle import c_oracle as C

    mp.start_processes(_worker, args=(WORLD, free_port(), str(tmp_path), case), nprocs=WORLD,
                       join=True, start_method="spawn")
    n, h, w, s, interp, reduce = case
    stack = np.random.default_rng(123).integers(0, 65536, (n, h, w)).astype(np.uint16)
    _, want = C.deskew(stack, s, interp, want_volume=False, reduce=reduce)
    got = np.load(tmp_path / "r0.npz")
    np.testing.assert_array_equal(got["xy"], want[0])
    np.testing.assert_array_equal(got["xz"], want[1])
    np.testing.assert_array_equal(got["yz"], want[2])
    assert int(got["disp_n"]) == WORLD


def test_plans_cover_scan_and_config5_windows():
    s45 = 0.7071067811865476
    plans = D.plan_slabs(8192, 2048, s45, "linear", 8)
    assert sum(p.count for p in plans) == 8192
    assert [p.first for p in plans] == [1024 * r for r in range(8)]
    assert all(p.canvas_rows == 7840 for p in plans)
    # each slab touches ~1024*s + H rows of the 7840-row canvas
    assert all(2770 <= p.u_count <= 2773 for p in plans)
    # the linear span floors, the canvas height ceils: the last canvas row can stay untouched
    assert plans[0].u_begin == 0 and plans[-1].u_begin + plans[-1].u_count in (7839, 7840)


def test_uneven_and_empty_slabs():
    plans = D.plan_slabs(3, 4, 1.0, "nearest", 5)
    assert [p.count for p in plans] == [1, 1, 1, 0, 0]
    assert D.shard_stacks(64, 3, 8) == [3, 11, 19, 27, 35, 43, 51, 59]


def _wrap_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plans = D.plan_slabs(4, 3, 1.0, "nearest", world)  # canvas rows 6
        p = plans[rank]
        part = np.full((p.u_count, 5), 0xFFFFFFF0 + rank, dtype=np.uint32)
        part[0, 0] = 7
        xy = D.combine_xy(torch.from_numpy(part), p, 5, "sum")
        if rank == 0:
            np.save(os.path.join(out_dir, "xy.npy"), xy.numpy())
            np.save(os.path.join(out_dir, "plans.npy"), np.array([[q.u_begin, q.u_count] for q in plans]))
    finally:
        dist.destroy_process_group()


def test_sum_combine_wraps_like_uint32(tmp_path):
    """uint32 sums travel bit-cast as int32: the merge equals uint32 addition mod 2^32."""
    mp.start_processes(_wrap_worker, args=(WORLD, free_port(), str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    got = np.load(tmp_path / "xy.npy")
    plans = np.load(tmp_path / "plans.npy")
    want = np.zeros((6, 5), dtype=np.uint64)
    for r, (b, c) in enumerate(plans):
        part = np.full((c, 5), 0xFFFFFFF0 + r, dtype=np.uint64)
        part[0, 0] = 7
        want[b:b + c] += part
    assert got.dtype == np.uint32
    np.testing.assert_array_equal(got, (want % (1 << 32)).astype(np.uint32))
    assert (want >= (1 << 32)).any()  # the case really wraps


def test_halo_planes_in_the_plan():
    """Slabs may carry halo input planes (north_star: scan-axis slabs with halo planes); they are
    clipped at the scan ends and never change which slices a rank owns."""
    plans = D.plan_slabs(100, 16, 0.7, "linear", 4, halo=3)
    assert [p.count for p in plans] == [25] * 4
    assert [(p.halo_lo, p.halo_hi) for p in plans] == [(0, 3), (3, 3), (3, 3), (3, 0)]
    assert [(p.in_first, p.in_count) for p in plans] == [(0, 28), (22, 31), (47, 31), (72, 28)]
    base = D.plan_slabs(100, 16, 0.7, "linear", 4)
    assert [(p.first, p.count, p.u_begin, p.u_count) for p in plans] == \
           [(p.first, p.count, p.u_begin, p.u_count) for p in base]
    with pytest.raises(ValueError):
        D.plan_slabs(10, 4, 1.0, "linear", 2, halo=-1)
