#!/bin/bash
# ncu evidence for the round: launch lists (device time per launch) and one --set full capture
# per key kernel.  Each ncu command runs only after the identical command exited 0 without ncu.
#   TAG=r01g bash scripts/profile_round.sh      -> gpurun_out/prof_$TAG/
set -u
TAG=${TAG:-r01}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
run() {   # name, command
  local name=$1; shift
  "$@" > $OUT/plain_$name.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_$name.csv "$@" \
      > $OUT/ncu_launch_$name.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:split_kv -s 3 -c 1 -o $OUT/full_$name "$@" \
      > $OUT/ncu_full_$name.log 2>&1 && \
    ncu -i $OUT/full_$name.ncu-rep --page raw --csv > $OUT/raw_$name.csv 2>/dev/null && \
    ncu -i $OUT/full_$name.ncu-rep --page details > $OUT/details_$name.txt 2>/dev/null
  local rc=$?
  # the exported pages are what is kept; the report itself only with KEEP_REP=1 (gpurun copies
  # back at most 64 MiB of gpurun_out/)
  [ "${KEEP_REP:-0}" = "1" ] || rm -f $OUT/full_$name.ncu-rep
  echo "$name rc=$rc"
}
# the headline (bench.py defaults: high_load, seq_aware_sm = s 1), the latency configs, and both
# long-context plans the bench's roofline_streaming times (the paper's rule s = 16 workspace, C-ext-1 s = 10)
run high_load python bench.py --steps 3 --warmup 3 --no-extras --cpu-seconds 1
run llama70b python bench.py --workload llama70b --steps 20 --warmup 3 --no-extras --cpu-seconds 1
run llama70b_tp8 python bench.py --workload llama70b_tp8 --steps 20 --warmup 3 --no-extras --cpu-seconds 1
run long_context python bench.py --workload long_context --policy seq_aware --steps 5 --warmup 3 --no-extras --cpu-seconds 1
run long_context_sm python bench.py --workload long_context --steps 5 --warmup 3 --no-extras --cpu-seconds 1
run mqa_g64 python bench.py --workload mqa_g64 --steps 5 --warmup 3 --no-extras --cpu-seconds 1
ls -la $OUT
