#!/bin/bash
# 8-byte-aligned rows (W = 2044): linear and nearest, volume + 3 MIPs and XY only
cd "$(dirname "$0")/.."
for i in linear nearest; do
  python tools/profile_run.py --iters 20 --w 2044 --interp $i
  python tools/profile_run.py --iters 20 --w 2044 --interp $i --no-volume --axes 0
  python tools/profile_run.py --iters 20 --w 2044 --interp $i --reduce sum
done
