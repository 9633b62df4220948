#!/bin/bash
# Quick iteration: GPU suite, smoke, attention micro-bench, short bench. Usage: bash tools/gpu_quick2.sh TAG [bench args]
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_$TAG.log
tail -3 $OUT/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
tail -2 $OUT/smoke_$TAG.log
timeout 300 python tools/attn_bench.py > $OUT/attn_$TAG.log 2>&1; cat $OUT/attn_$TAG.log | tail -8
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline "$@" > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
tail -1 $OUT/bench_$TAG.err
python tools/bench_brief.py $OUT/bench_$TAG.json
