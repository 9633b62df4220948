#!/bin/bash
# Round-2 re-entry check: GPU suite, smoke, default bench (driver-equivalent).
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_j.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_j.log
tail -5 $OUT/pytest_gpu_j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke_j.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_j.log
tail -3 $OUT/smoke_j.log
timeout 900 python bench.py > $OUT/bench_j.json 2> $OUT/bench_j.err; echo "bench exit $?" >> $OUT/bench_j.err
tail -3 $OUT/bench_j.err
python -c "import json; b=json.load(open('$OUT/bench_j.json')); print('value', b['value'], 'TTFT', b['ttft_p50_ms'], 'e2e', b['e2e'], 'frac', b['roofline']['frac'])"
