#!/bin/bash
# one ncu --set full capture: bash tools/gpu_ncu1.sh TAG REGEX SKIP COUNT [profile_step args]
TAG=$1; RE=$2; SKIP=$3; CNT=$4; shift 4
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:$RE -s $SKIP -c $CNT -o gpurun_out/prof_$TAG -f python tools/profile_step.py "$@" > gpurun_out/prof_$TAG.log 2>&1
tail -2 gpurun_out/prof_$TAG.log
