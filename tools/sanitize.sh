#!/bin/bash
# compute-sanitizer over the driver smoke (bf16 tcgen05 restore, coded store,
# decode + K1 fold, K3 selector) and the f32 turn-loop parity test:
# memcheck, racecheck (shared-memory hazards), synccheck (barrier misuse).
# Usage: bash tools/sanitize.sh TAG   (logs -> gpurun_out/sanitize_TAG_*.log)
TAG=${1:-r02}
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 3 \
    python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitize_${TAG}_smoke_$tool.log 2>&1
  echo "smoke $tool exit $?" | tee -a $OUT/sanitize_${TAG}_smoke_$tool.log
  tail -2 $OUT/sanitize_${TAG}_smoke_$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 3 \
  python -m pytest tests/test_gpu_turns.py -x -q -k "bit_exact and 0" > $OUT/sanitize_${TAG}_turns_memcheck.log 2>&1
echo "turns memcheck exit $?" | tee -a $OUT/sanitize_${TAG}_turns_memcheck.log
tail -2 $OUT/sanitize_${TAG}_turns_memcheck.log
