#!/bin/bash
# side-projection sweep plus the sum-mode variants that share the XZ staging buffer
cd "$(dirname "$0")/.."
tools/time_side.sh
python tools/profile_run.py --iters 20 --reduce sum
python tools/profile_run.py --iters 20 --no-volume --reduce sum
