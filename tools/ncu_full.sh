#!/bin/bash
# ncu --set full capture of one step-kernel launch: tools/ncu_full.sh <config> <fast|exact> <tag>
cfg=$1; mode=$2; tag=$3
CMD="python tools/prof_step.py $cfg 4 $([ "$mode" = fast ] && echo fast)"
timeout 120 $CMD > gpurun_out/plain_$tag.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swe_step_kernel -s 2 -c 1 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
