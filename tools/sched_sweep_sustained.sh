#!/bin/bash
# Sustained (power-capped) bench.py A/B of scheduler knobs given as env assignments, interleaved.
#   tools/sched_sweep_sustained.sh REPS "" "SSB_TAIL_ITEMS_PER_CTA=3" ...
cd "$(dirname "$0")/.."
reps=$1; shift
for rep in $(seq "$reps"); do
  for cfg in "$@"; do
    env $cfg python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${cfg:-default}', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])"
  done
done
