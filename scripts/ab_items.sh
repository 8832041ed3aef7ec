#!/bin/bash
# A/B of the work-item size (DECATTN_ITEM_BLOCKS) on latency and streaming workloads, interleaved.
# usage: bash scripts/ab_items.sh <rounds> <lib>...
R=$1; shift
us() { python -c "import json,sys; print(json.loads(sys.stdin.read())['us_per_step'])"; }
for r in $(seq $R); do
  for L in "$@"; do
    a=$(DECATTN_LIB=$L python bench.py --workload llama70b --no-extras --steps 200 2>/dev/null | us)
    b=$(DECATTN_LIB=$L python bench.py --workload llama70b_tp8 --no-extras --steps 200 2>/dev/null | us)
    c=$(DECATTN_LIB=$L python bench.py --workload llama70b --policy guarded --no-extras --steps 200 2>/dev/null | us)
    d=$(DECATTN_LIB=$L python bench.py --workload high_load --no-extras --steps 10 2>/dev/null | us)
    e=$(DECATTN_LIB=$L python bench.py --workload long_context --no-extras --steps 20 2>/dev/null | us)
    echo "$(basename $L) llama $a tp8 $b llama_guarded $c high_load $d long $e"
  done
done
