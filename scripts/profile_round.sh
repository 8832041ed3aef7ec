#!/bin/bash
# ncu evidence for the round: launch lists (device time per launch) and one --set full capture
# per key kernel.  Each ncu command runs only after the identical command exited 0 without ncu.
set -u
OUT=gpurun_out
CMD_LLAMA="python bench.py --steps 20 --warmup 3 --no-extras --cpu-seconds 1"
CMD_TP8="python bench.py --workload llama70b_tp8 --steps 20 --warmup 3 --no-extras --cpu-seconds 1"
CMD_HL="python bench.py --workload high_load --steps 3 --warmup 3 --no-extras --cpu-seconds 1"
$CMD_LLAMA > $OUT/plain_llama.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_llama70b.csv $CMD_LLAMA > $OUT/ncu_launch_llama.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:split_kv -s 3 -c 1 -o $OUT/prof_llama70b $CMD_LLAMA > $OUT/ncu_full_llama.log 2>&1
echo "llama rc=$?"
$CMD_TP8 > $OUT/plain_tp8.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_tp8.csv $CMD_TP8 > $OUT/ncu_launch_tp8.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:split_kv -s 3 -c 1 -o $OUT/prof_tp8 $CMD_TP8 > $OUT/ncu_full_tp8.log 2>&1
echo "tp8 rc=$?"
$CMD_HL > $OUT/plain_hl.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:split_kv -s 2 -c 1 -o $OUT/prof_high_load $CMD_HL > $OUT/ncu_full_hl.log 2>&1
echo "high_load rc=$?"
ls -la $OUT
