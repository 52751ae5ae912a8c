"""bench.py's JSON contract, checked on CPU through the reference arm (no GPU needed).

The driver parses one JSON line per run; the reference arm (`--impl reference`) times the
reference algorithm's CPU port and must print the same keys as the GPU arm plus
``impl`` / ``cpu_baseline`` / ``e2e``.  Ranks other than 0 print nothing and exit 0.
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                          cwd=REPO, env=e, timeout=600)


def test_reference_arm_prints_one_contract_line():
    r = run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1", "--ref-seconds", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("config1")


def test_reference_arm_nonzero_ranks_exit_quietly():
    r = run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1", "--ref-seconds", "1"],
            env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]


def test_reference_arm_is_bounded_for_many_steps():
    # the driver may pass a large --steps K: the per-step sample shrinks so the run stays short
    import time

    t0 = time.perf_counter()
    r = run(["--impl", "reference", "--config", "1", "--steps", "40", "--warmup", "3"])
    wall = time.perf_counter() - t0
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")][-1])
    assert d["steps"] == 40 and d["value"] > 0
    assert wall < 240, wall


def test_reference_arm_config_matches_ours():
    # same config keys as the GPU arm (the driver compares them field by field)
    r = run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1", "--ref-seconds", "1"])
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")][-1])
    for k in ("workload", "interp", "shear_px", "canvas", "outputs"):
        assert k in d["config"], k
    # ms_per_step is one full stack's worth of reference work
    n, (u, w) = 128, d["config"]["canvas"]
    assert abs(d["ms_per_step"] - n * u * w / (d["value"] * 1e9) * 1e3) < 1e-6 * d["ms_per_step"]


def test_gpus_n_self_launches_n_ranks_dry_run():
    # `bench.py --gpus N` without torchrun re-executes itself with N ranks (gloo on CPU here)
    for n in (2, 3):
        r = run(["--gpus", str(n), "--dry-run", "--backend", "gloo", "--steps", "3", "--warmup", "3"])
        assert r.returncode == 0, r.stderr[-2000:]
        lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
        assert len(lines) == 1, r.stdout
        d = json.loads(lines[0])
        assert d["n_gpus"] == n and d["dry_run"] is True and d["value"] is None
        assert d["config"]["workload"].startswith("config4") and d["config"]["display_gather_ok"] is True
        assert d["config"]["stacks_per_rank"] == len(range(0, 64, n))
