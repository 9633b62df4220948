mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "estimator or turn_loop or decode" > gpurun_out/pytest_r2f.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2f.log; tail -3 gpurun_out/pytest_r2f.log
for v in base new; do
  if [ $v = base ]; then export KRUL_LIB=alt_lib/r2_base/libkrul_b200.so; else unset KRUL_LIB; fi
  timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_r2f_$v.json 2> gpurun_out/bench_r2f_$v.err
  python - <<PY
import json
b=json.load(open('gpurun_out/bench_r2f_$v.json'))
r=b['rooflines']
print('$v', 'TTFT', b['ttft_p50_ms'], 'rc', b['config']['r_c'], 'h2d', b['restore']['h2d_ms'], 'dx', r.get('decode_expand',b['roofline']).get('avg_launch_us'), 'fold', r['estimator_decode_fold'])
PY
done
