#!/bin/bash
# A/B library builds on the streaming workloads: bash scripts/ab_stream.sh <lib>... (interleaved, 2 rounds)
for r in 1 2; do
  for L in "$@"; do
    for w in high_load long_context; do
      st=5; [ $w = long_context ] && st=20
      DECATTN_LIB=$L python bench.py --workload $w --no-extras --steps $st 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L) $w', d['us_per_step'], d['value'])"
    done
  done
done
