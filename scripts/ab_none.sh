#!/bin/bash
# A/B no-combine (s = 1) kernel configurations: streaming (high-load) and latency (guarded Llama s = 1)
for r in 1 2; do
  for L in "$@"; do
    a=$(DECATTN_LIB=$L python bench.py --workload high_load --no-extras --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_step'])")
    b=$(DECATTN_LIB=$L python bench.py --policy guarded --no-extras --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_step'])")
    c=$(DECATTN_LIB=$L python bench.py --workload llama70b_tp8 --policy guarded --no-extras --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_step'])")
    echo "$(basename $L) high_load $a  llama_guarded $b  tp8_guarded $c"
  done
done
