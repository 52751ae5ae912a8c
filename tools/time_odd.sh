#!/bin/bash
# odd-width timings (config-2 shape, W = 2044 / 2046 / 2047): volume + 3 MIPs, XY only, 3 MIPs
cd "$(dirname "$0")/.."
for w in 2044 2046 2047; do
  python tools/profile_run.py --iters 20 --w $w
  python tools/profile_run.py --iters 20 --w $w --no-volume --axes 0
  python tools/profile_run.py --iters 20 --w $w --no-volume
done
