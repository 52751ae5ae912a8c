#!/bin/bash
# Sum-mode timing sweep (config 2 shapes)
cd "$(dirname "$0")/.."
python tools/profile_run.py --iters 20 --reduce sum
python tools/profile_run.py --iters 20 --reduce sum --no-volume
python tools/profile_run.py --iters 20 --reduce sum --interp nearest
