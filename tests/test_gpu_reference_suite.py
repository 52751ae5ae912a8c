"""The reference's own test suite, run unmodified against the drop-in.

``baseline/_ref`` holds the unmodified reference package and its test files
(``baseline/install_ref.sh``; git-ignored, it travels to the GPU box).  A pytest subprocess runs
those files with ``tests/reference_shim.py``, which swaps the reference's hot path for the drop-in:
``ProjectionCanvas`` / ``deskew_place`` / ``warp_projection`` (ss/pipeline.py) and
``reference_deskew`` (ss/phantom.py).  That covers the hand examples and properties of
pkg/tests/test_pipeline.py:107-304, test_phantom.py:233-324, test_acceptance.py:95-171, the
``LivePipeline`` tests of test_pipeline.py:469-630 (canvas per channel, mode and view changes,
rolling-mode ``max_pixels.copy()``) and ``cli.run_batch`` (test_cli.py) on the GPU canvas.
"""

import os
import re
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF_TESTS = os.path.join(REPO, "baseline", "_ref", "ref_tests")

pytestmark = pytest.mark.gpu

# test files that reach the deskew path (server / source / geometry / bench run reference code only,
# but go along: a shim that broke an import anywhere would show up there)
FILES = ["test_pipeline.py", "test_phantom.py", "test_acceptance.py", "test_cli.py", "test_bench.py",
         "test_server.py", "test_source.py", "test_geometry.py"]


# wall-clock-ordinal tests of the reference's stage-cost analytics (flaky under
# load even on the reference itself); they time CPU stages, not the deskew path's results
FLAKY = ["test_acceptance.py::test_stage_cost_scaling_table_and_crossover_order"]


def run_suite(files, extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([HERE, REPO, os.path.join(REPO, "baseline", "_ref"), env.get("PYTHONPATH", "")])
    deselect = [a for t in FLAKY for a in ("--deselect", os.path.join(REF_TESTS, t))]
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "reference_shim", "-rfE",
           *deselect, *extra, *[os.path.join(REF_TESTS, f) for f in files]]
    return subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1800)


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not installed (baseline/install_ref.sh)")
def test_reference_suite_passes_on_drop_in():
    r = run_suite(FILES)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", "reference_suite_on_drop_in.txt"), "w") as f:
        f.write(out)
    assert r.returncode == 0, out[-6000:]
    assert "CANVAS=paper_2211_00645_b200.pipeline" in out  # the shim was active
    launches = int(re.search(r"SSB_LAUNCHES=(\d+)", out).group(1))
    assert launches > 1000, launches  # the device canvas did the work
    assert re.search(r"(\d+) passed", out)
