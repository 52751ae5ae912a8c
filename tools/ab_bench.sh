#!/bin/bash
# Sustained (power-capped) A/B of library variants through bench.py: interleaved, 2 reps each.
cd "$(dirname "$0")/.."
cp paper_2211_00645_b200/lib/libssb.so /tmp/libssb_orig.so
for v in "$@"; do
  cp "variants/libssb_$v.so" paper_2211_00645_b200/lib/libssb.so
  echo "== $v parity: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
done
for rep in 1 2; do
  for v in "$@"; do
    cp "variants/libssb_$v.so" paper_2211_00645_b200/lib/libssb.so
    python bench.py --no-e2e --no-cpu-baseline "${BENCH_ARGS[@]}" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'rep $rep', round(d['ms_per_step'],4), 'ms', round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],3), d['clocks'])"
  done
done
cp /tmp/libssb_orig.so paper_2211_00645_b200/lib/libssb.so
