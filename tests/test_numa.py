"""NUMA placement helper of the pinned H2D pipeline (stream.near_gpu), host logic only."""
import os

from paper_2211_00645_b200 import stream


def test_parse_cpulist():
    assert stream._parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert stream._parse_cpulist("5") == {5}
    assert stream._parse_cpulist("") == set()


def test_near_gpu_restores_affinity_without_a_gpu():
    before = os.sched_getaffinity(0)
    with stream.near_gpu(None):
        pass
    assert os.sched_getaffinity(0) == before


def test_near_gpu_restores_affinity_when_bound(monkeypatch):
    before = os.sched_getaffinity(0)
    one = {min(before)}
    monkeypatch.setattr(stream, "gpu_numa_cpus", lambda device=None: one)
    with stream.near_gpu(None):
        assert os.sched_getaffinity(0) == one
    assert os.sched_getaffinity(0) == before
