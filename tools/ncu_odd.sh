#!/bin/bash
# ncu of the odd-width live view (W = 2044, XY only: row-class TMA with lane-31 boxes), summarised on the box
cd "$(dirname "$0")/.."
python tools/profile_run.py --iters 1 --w 2044 --no-volume --axes 0 > /dev/null 2>&1 || exit 1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:deskew_tma -c 1 -o /tmp/w2044xy \
  python tools/profile_run.py --iters 1 --w 2044 --no-volume --axes 0 > gpurun_out/ncu_w2044xy.log 2>&1
python tools/ncu_summary.py /tmp/w2044xy.ncu-rep > gpurun_out/final_w2044xy_ncu_summary.txt 2>&1
ncu -i /tmp/w2044xy.ncu-rep --page source --csv --print-source sass > /tmp/w2044xy.csv 2>/dev/null
python tools/sass_mix.py /tmp/w2044xy.csv 25 >> gpurun_out/final_w2044xy_ncu_summary.txt 2>&1
rm -f /tmp/w2044xy.ncu-rep /tmp/w2044xy.csv
