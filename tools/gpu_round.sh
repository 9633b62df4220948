#!/bin/bash
# One gpurun call: GPU parity suite, smoke, bench, launch list, ncu capture of the top kernel.
# Usage (from repo root on the box): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $OUT/launches_$TAG.csv python tools/profile_step.py > $OUT/launches_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:${KERNEL:-k_gemm_tc} -c ${NCAP:-3} -o $OUT/prof_$TAG -f python tools/profile_step.py > $OUT/prof_$TAG.log 2>&1
echo done
