#!/bin/bash
# Timing sweep of the max-mode side-projection variants (config 2 shapes): projection-only
# 3 MIPs / XY+XZ / XY+YZ / XY only, and the headline volume + 3 MIPs.
cd "$(dirname "$0")/.."
python tools/profile_run.py --iters 20 --no-volume
python tools/profile_run.py --iters 20 --no-volume --axes 0,1
python tools/profile_run.py --iters 20 --no-volume --axes 0,2
python tools/profile_run.py --iters 20 --no-volume --axes 0
python tools/profile_run.py --iters 20
