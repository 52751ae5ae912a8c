#!/bin/bash
# Install the unmodified reference (skewstream, /root/reference/pkg) into baseline/_ref, plus a copy of
# its own test files in baseline/_ref/ref_tests.  baseline/_ref is git-ignored but travels to the GPU
# box with gpurun, where tests/test_gpu_reference_suite.py runs those files with the hot path swapped
# for the drop-in (tests/reference_shim.py).  Run in the build container (the only place
# /root/reference exists); the source tree is read-only, so pip builds from a copy.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/ssref && cp -r /root/reference/pkg /tmp/ssref && chmod -R u+w /tmp/ssref
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps --upgrade \
    --target baseline/_ref /tmp/ssref
rm -rf baseline/_ref/ref_tests && cp -r /tmp/ssref/tests baseline/_ref/ref_tests
echo "reference installed: $(ls baseline/_ref)"
