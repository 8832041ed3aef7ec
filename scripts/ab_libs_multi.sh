#!/bin/bash
# A/B several library builds on the latency shapes, interleaved: bash scripts/ab_libs_multi.sh <rounds> <lib>...
R=$1; shift
for r in $(seq $R); do
  for L in "$@"; do
    a=$(DECATTN_LIB=$L python bench.py --workload llama70b --no-extras --steps 200 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['us_per_step'])")
    b=$(DECATTN_LIB=$L python bench.py --workload llama70b_tp8 --no-extras --steps 200 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['us_per_step'])")
    c=$(DECATTN_LIB=$L python bench.py --workload llama70b --policy guarded --no-extras --steps 200 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['us_per_step'])")
    echo "$(basename $L) llama $a  tp8 $b  llama_guarded $c"
  done
done
