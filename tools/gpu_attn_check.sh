timeout 300 python -m pytest tests -m gpu -q -x -k "attention or restore or prefill" 2>&1 | tail -1
for i in 1 2 3; do timeout 300 python -m pytest tests -m gpu -q -x -k "tcgen05_attention" 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k_attn_fa --csv --log-file gpurun_out/attn_ts.csv python tools/profile_step.py --rc 0.068 > /dev/null 2>&1
KRUL_ATTN_STRICT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k_attn_fa --csv --log-file gpurun_out/attn_ts_strict.csv python tools/profile_step.py --rc 0.068 > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-policies > gpurun_out/bench_g24.json 2>/dev/null
