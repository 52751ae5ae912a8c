#!/bin/bash
# ncu of the projection-only 3-MIP live view (config-2 shape), summarised on the box
cd "$(dirname "$0")/.."
python tools/profile_run.py --iters 1 --no-volume > /dev/null 2>&1 || exit 1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:deskew_tma -c 1 -o /tmp/mip3 \
  python tools/profile_run.py --iters 1 --no-volume > gpurun_out/ncu_mip3.log 2>&1
python tools/ncu_summary.py /tmp/mip3.ncu-rep > gpurun_out/final_mip3_staged_ncu_summary.txt 2>&1
ncu -i /tmp/mip3.ncu-rep --page source --csv --print-source sass > /tmp/mip3.csv 2>/dev/null
python tools/sass_mix.py /tmp/mip3.csv 25 >> gpurun_out/final_mip3_staged_ncu_summary.txt 2>&1
rm -f /tmp/mip3.ncu-rep /tmp/mip3.csv
