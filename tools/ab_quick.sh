#!/bin/bash
# Quick A/B of prebuilt variants (variants/libssb_<name>.so): a bounded parity subset per variant
# (PARITY="pytest args", default the batch + parity files), then interleaved timing (TIMER script).
cd "$(dirname "$0")/.."
cp paper_2211_00645_b200/lib/libssb.so /tmp/libssb_orig.so
for v in "$@"; do
  cp "variants/libssb_$v.so" paper_2211_00645_b200/lib/libssb.so
  echo "== $v parity: $(timeout ${PTIME:-240} python -m pytest ${PARITY:-tests/test_gpu_batch.py tests/test_gpu_parity.py} -m gpu -x -q 2>&1 | tail -1)"
done
for rep in 1 2; do
  for v in "$@"; do
    cp "variants/libssb_$v.so" paper_2211_00645_b200/lib/libssb.so
    echo "== $v (rep $rep)"
    timeout 120 ${TIMER:-tools/time_variants.sh}
  done
done
cp /tmp/libssb_orig.so paper_2211_00645_b200/lib/libssb.so
