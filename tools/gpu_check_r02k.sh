#!/bin/bash
# TMA-staged k_expand: GPU suite, smoke, default bench, raw-store bench, ncu of k_expand.
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_k.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_k.log
tail -4 $OUT/pytest_gpu_k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke_k.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_k.log
tail -2 $OUT/smoke_k.log
timeout 900 python bench.py > $OUT/bench_k.json 2> $OUT/bench_k.err; echo "bench exit $?" >> $OUT/bench_k.err
tail -1 $OUT/bench_k.err
python -c "import json; b=json.load(open('$OUT/bench_k.json')); print('value', b['value'], 'TTFT', b['ttft_p50_ms'], 'e2e', b['e2e']['value'], 'frac', b['roofline']['frac'], 'policies', {k: v['ttft_ms'] for k, v in b['policies'].items()})"
KRUL_KV_CODING=0 timeout 900 python bench.py --steps 10 --no-cpu-baseline > $OUT/bench_k_raw.json 2> $OUT/bench_k_raw.err; echo "raw bench exit $?" >> $OUT/bench_k_raw.err
tail -1 $OUT/bench_k_raw.err
python -c "import json; b=json.load(open('$OUT/bench_k_raw.json')); print('raw value', b['value'], 'TTFT', b['ttft_p50_ms'], 'restore', b['restore'], {k: (v.get('frac'), v.get('avg_launch_us'), v.get('achieved')) for k, v in b['rooflines'].items() if isinstance(v, dict)})"
KRUL_KV_CODING=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_expand -c 8 --csv \
  --log-file $OUT/ncu_expand_k.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_expand_k.log 2>&1; echo "ncu exit $?"
head -30 $OUT/ncu_expand_k.csv
