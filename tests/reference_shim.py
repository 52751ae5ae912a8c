"""pytest plugin: the reference's own test files, with its hot path swapped for the drop-in.

Loaded with ``-p reference_shim`` by ``tests/test_gpu_reference_suite.py`` (GPU box), this does what
INTEGRATION.md's switch-over shim does inside ``skewstream``: every entry point on the deskew path
resolves to ``paper_2211_00645_b200`` -- ``ProjectionCanvas`` (canvas in HBM, fused sm_100a kernels),
``deskew_place``, ``warp_projection`` (ss/pipeline.py:239-457) and ``phantom.reference_deskew``
(ss/phantom.py:359-402) -- and the drop-in's exceptions become subclasses of the reference's
(``errors.adopt``).  Everything that constructs a canvas picks it up unchanged: ``LivePipeline``
(ss/pipeline.py:677-1064, including mode / view changes and rolling-mode ``max_pixels.copy()``),
``cli.run_batch`` (ss/cli.py:308-338) and ``bench`` (ss/bench.py, which binds the names at import).
The reference package comes from ``baseline/_ref`` (``baseline/install_ref.sh``), never from
``/root/reference``.  Test infrastructure only; the product does not import this.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = os.path.join(REPO, "baseline", "_ref")
for p in (REF, REPO):
    if p not in sys.path:
        sys.path.insert(0, p)

import skewstream.bench as ref_bench  # noqa: E402
import skewstream.errors as ref_errors  # noqa: E402
import skewstream.phantom as ref_phantom  # noqa: E402
import skewstream.pipeline as ref_pipeline  # noqa: E402

from paper_2211_00645_b200 import errors, phantom, pipeline  # noqa: E402

SWAPPED = []


def _swap(module, name, value):
    setattr(module, name, value)
    SWAPPED.append(f"{module.__name__}.{name}")


errors.adopt(ref_errors)
for _name in ("ProjectionCanvas", "deskew_place", "warp_projection"):
    _swap(ref_pipeline, _name, getattr(pipeline, _name))
_swap(ref_phantom, "reference_deskew", phantom.reference_deskew)
for _name in ("ProjectionCanvas", "warp_projection"):  # bound by name at import (ss/bench.py:43)
    _swap(ref_bench, _name, getattr(pipeline, _name))


def pytest_report_header(config):
    return ["reference hot path swapped for the drop-in: " + ", ".join(SWAPPED)]


def pytest_sessionfinish(session, exitstatus):
    # prove the device path ran: the library's launch counter, printed for the calling test
    from paper_2211_00645_b200 import _lib

    print(f"\nSSB_LAUNCHES={_lib.launch_count()} CANVAS={ref_pipeline.ProjectionCanvas.__module__} "
          f"SWAPPED={','.join(SWAPPED)}")
