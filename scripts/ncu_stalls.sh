#!/bin/bash
# dense PC sampling of the latency-path kernels (TP-8 slice: guarded s=1 and seq-aware s=3)
set -u
CMD="python scripts/probe_one.py"
$CMD > gpurun_out/plain_probe_one.log 2>&1 && \
ncu --set full --warp-sampling-interval 0 --warp-sampling-max-passes 20 --clock-control none --import-source on -k regex:split_kv -s 40 -c 2 -o gpurun_out/stalls $CMD > gpurun_out/ncu_stalls.log 2>&1
echo rc=$?
