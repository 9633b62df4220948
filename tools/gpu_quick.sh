#!/bin/bash
# Quick gpurun iteration: GPU tests, bench, launch list. Usage: bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
if [ -n "$2" ]; then K="-k $2"; fi
timeout 900 python -m pytest tests -m gpu -x -q $K > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
tail -15 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
tail -3 $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file $OUT/launches_$TAG.csv python tools/profile_step.py > $OUT/launches_$TAG.log 2>&1
python tools/ncu_summary.py --launches $OUT/launches_$TAG.csv | head -14
python -c "import json; b=json.load(open('$OUT/bench_$TAG.json')); print('TTFT', b['ttft_p50_ms'], 'rc', b['config']['r_c'], b['restore'], b['roofline'])"
