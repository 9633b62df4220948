#!/bin/bash
# Attention iteration: parity tests touching attention, micro-bench + timeline in both wait modes.
TAG=$1; OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "attn or attention or fa or prefill or restore" > $OUT/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_$TAG.log
tail -2 $OUT/pytest_$TAG.log
for sl in 1 0; do
  echo "== KRUL_ATTN_SLEEP=$sl"
  KRUL_ATTN_SLEEP=$sl timeout 300 python tools/attn_bench.py 2>&1 | tail -8
  KRUL_ATTN_SLEEP=$sl timeout 300 python tools/attn_timeline.py 128 8192 0 128 8192 32 1024 0 0 2>&1 | tail -30
done
