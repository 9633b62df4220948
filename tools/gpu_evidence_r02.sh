#!/bin/bash
# Round-2 evidence pass: GPU suite, smoke, default bench (as the driver runs
# it), reference arm, ncu launch list, ncu --set full of the top kernels.
TAG=${1:-r02}; OUT=gpurun_out; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py --gpus 1 --steps 50 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 2 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref exit $?" >> $OUT/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $OUT/launches_$TAG.csv python tools/profile_step.py --rc 0.02 > $OUT/launches_$TAG.log 2>&1
cap() {  # name regex skip count rc
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"$2" -s $3 -c $4 -o $OUT/prof_$1_$TAG -f python tools/profile_step.py --rc $5 > $OUT/prof_$1_$TAG.log 2>&1
}
# the new-input prefill's kernels (r_c = 0: no pyramid launches in between)
cap gstream '^k_gemm_tc$' 40 4 0.0
cap attn 'k_attn_fa' 20 1 0.0
cap comb 'k_attn_combine' 20 1 0.0
cap dexp 'k_ec_decode_expand' 10 1 0.0
cap logits 'k_logits' 0 1 0.0
# the pyramid recompute's CTA-pair GEMMs
cap gemm '^k_gemm_tc2$' 0 2 0.1
# the K1 decode fold (32 layers x 32 heads x W 8328) alone: one --set full
# capture, the per-CTA timeline and graph-replayed device time
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fold_direct -c 1 \
    -o $OUT/prof_fold_$TAG -f python tools/fold_bench.py > $OUT/prof_fold_$TAG.log 2>&1
FOLD_TIMELINE=1 FOLD_LOOP=200 timeout 300 python tools/fold_bench.py > $OUT/fold_$TAG.txt 2>&1
timeout 120 ./tools/exp/fp2_rate > $OUT/fp2_rate_$TAG.txt 2>&1
bash tools/sanitize.sh $TAG
echo done
