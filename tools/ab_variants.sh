#!/bin/bash
# A/B timing of prebuilt library variants (variants/libssb_<name>.so), interleaved.
# usage: tools/ab_variants.sh name1 name2 ...   (run on the GPU box)
set -e
cd "$(dirname "$0")/.."
cp paper_2211_00645_b200/lib/libssb.so /tmp/libssb_orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp "variants/libssb_$v.so" paper_2211_00645_b200/lib/libssb.so
    echo "== $v (rep $rep)"
    python tools/profile_run.py --iters 20
    python tools/profile_run.py --iters 20 --no-volume
    python tools/profile_run.py --iters 20 --no-volume --axes 0
    python tools/profile_run.py --iters 20 --reduce sum
    python tools/profile_run.py --iters 20 --interp nearest
  done
done
cp /tmp/libssb_orig.so paper_2211_00645_b200/lib/libssb.so
