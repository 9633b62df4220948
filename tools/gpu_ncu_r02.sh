#!/bin/bash
# ncu --set full captures of the step's top kernels (one launch each) at r_c = RC.
TAG=${1:-r02}; OUT=gpurun_out; mkdir -p $OUT; RC=${RC:-0.0}
cap() {  # name regex skip count
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"$2" -s $3 -c $4 -o $OUT/prof_$1_$TAG -f python tools/profile_step.py --rc $RC > $OUT/prof_$1_$TAG.log 2>&1
  tail -1 $OUT/prof_$1_$TAG.log
}
cap attn 'k_attn_fa' 20 1
cap comb 'k_attn_combine' 20 1
cap dexp 'k_ec_decode_expand' 10 1
cap gstream '^k_gemm_tc$' 40 4
cap norm 'k_rmsnorm' 20 1
echo done
