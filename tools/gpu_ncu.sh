#!/bin/bash
# ncu --set full captures of selected kernels of one restore+prefill step.
# Usage: bash tools/gpu_ncu.sh TAG "regex1:count1 regex2:count2 ..."
TAG=${1:-n}
OUT=gpurun_out
mkdir -p $OUT
i=0
for spec in $2; do
  re=${spec%%:*}; cnt=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:$re -c $cnt -o $OUT/prof_${TAG}_$i -f python tools/profile_step.py > $OUT/prof_${TAG}_$i.log 2>&1
  tail -2 $OUT/prof_${TAG}_$i.log
  i=$((i+1))
done
