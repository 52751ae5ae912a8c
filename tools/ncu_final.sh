#!/bin/bash
# ncu captures summarised on the box (the .ncu-rep files are removed: gpurun_out must stay < 64 MiB)
cd "$(dirname "$0")/.."
cap() {  # name, profile_run args
  local name=$1; shift
  python tools/profile_run.py --iters 1 "$@" > /dev/null 2>&1 || return
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:deskew_tma -c 1 -o /tmp/$name \
    python tools/profile_run.py --iters 1 "$@" > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep > gpurun_out/${name}_ncu_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.csv 2>/dev/null
  python tools/sass_mix.py /tmp/$name.csv 25 >> gpurun_out/${name}_ncu_summary.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/$name.csv
}
cap headline
cap mip3 --no-volume
cap xymax --no-volume --axes 0
cap w2044 --w 2044
cap w2047xy --w 2047 --no-volume --axes 0
