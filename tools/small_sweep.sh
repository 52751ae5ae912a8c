#!/bin/bash
# Scheduler knobs on a small stack (config 1: 128 x 256 x 512): items per CTA (phase 1 / tail), big-phase share
cd "$(dirname "$0")/.."
for a in "2 6" "1 2" "1 1" "1 0" "4 4"; do set -- $a; for pct in 85 100; do
  echo "per_cta=$1 tail=$2 pct=$pct $(SSB_ITEMS_PER_CTA=$1 SSB_TAIL_ITEMS_PER_CTA=$2 SSB_BIG_PERCENT=$pct python tools/profile_run.py --iters 50 --n 128 --h 256 --w 512 2>/dev/null)"
done; done
