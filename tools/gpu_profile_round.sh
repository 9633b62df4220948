#!/bin/bash
# Evidence pass: full bench (with CPU baseline), reference arm, launch list,
# ncu --set full of the top kernels. Usage: bash tools/gpu_profile_round.sh TAG
TAG=${1:-r}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
RC=${RC:-0.0}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $OUT/launches_$TAG.csv python tools/profile_step.py --rc $RC > $OUT/launches_$TAG.log 2>&1
# top kernels of the step: the new-input prefill's weight-streaming GEMMs (QKV, O, FFN1, FFN2 of
# layer 0), a new-prefill attention, a blob decode, an expand, the logits GEMV
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:^k_gemm_tc$ -c 4 -o $OUT/prof_gstream_$TAG -f python tools/profile_step.py --rc $RC > $OUT/prof_gstream_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_attn_fa -s 20 -c 1 -o $OUT/prof_attn_$TAG -f python tools/profile_step.py --rc $RC > $OUT/prof_attn_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_ec_decode -s 10 -c 1 -o $OUT/prof_decode_$TAG -f python tools/profile_step.py --rc $RC > $OUT/prof_decode_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_expand -s 10 -c 1 -o $OUT/prof_expand_$TAG -f python tools/profile_step.py --rc $RC > $OUT/prof_expand_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_logits -c 1 -o $OUT/prof_logits_$TAG -f python tools/profile_step.py --rc $RC > $OUT/prof_logits_$TAG.log 2>&1
# the recompute's pair GEMMs at the r_c the raw store would use
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_gemm_tc2 -c 3 -o $OUT/prof_gemm_$TAG -f python tools/profile_step.py --rc 0.068 > $OUT/prof_gemm_$TAG.log 2>&1
echo done
