#!/bin/bash
# A/B two builds of the library on the headline shapes, interleaved: bash scripts/ab_libs.sh <libA> <libB> [rounds]
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for L in $A $B; do
    for w in llama70b llama70b_tp8; do
      DECATTN_LIB=$L python bench.py --workload $w --no-extras --steps 200 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L) $w', d['us_per_step'])"
    done
  done
done
