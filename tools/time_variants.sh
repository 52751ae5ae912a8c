#!/bin/bash
# Timing sweep of the fused kernel over the main output variants (config 2 shapes).
cd "$(dirname "$0")/.."
python tools/profile_run.py --iters 20
python tools/profile_run.py --iters 20 --no-volume
python tools/profile_run.py --iters 20 --no-volume --axes 0
python tools/profile_run.py --iters 20 --reduce sum
python tools/profile_run.py --iters 20 --interp nearest
python tools/profile_run.py --iters 20 --no-volume --axes 0 --reduce sum --alpha 45
