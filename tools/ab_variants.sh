#!/bin/bash
# A/B of prebuilt library variants (variants/libssb_<name>.so): GPU parity suite once per
# variant, then interleaved timing sweeps (tools/time_variants.sh).   usage: tools/ab_variants.sh a b ...
cd "$(dirname "$0")/.."
cp paper_2211_00645_b200/lib/libssb.so /tmp/libssb_orig.so
for v in "$@"; do
  cp "variants/libssb_$v.so" paper_2211_00645_b200/lib/libssb.so
  echo "== $v parity: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
done
for rep in 1 2; do
  for v in "$@"; do
    cp "variants/libssb_$v.so" paper_2211_00645_b200/lib/libssb.so
    echo "== $v (rep $rep)"
    ${TIMER:-tools/time_variants.sh}
  done
done
cp /tmp/libssb_orig.so paper_2211_00645_b200/lib/libssb.so
