timeout 900 python -m pytest tests/test_gpu_batch.py tests -m gpu -x -q -k "attn or attention or batch or span or restore" 2>&1 | tail -2
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 3 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_race_fix.log 2>&1; echo "racecheck exit $?"; tail -2 gpurun_out/sanitize_race_fix.log
python tools/attn_bench.py 2>&1 | grep "target=0"
