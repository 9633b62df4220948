mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pdl.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_pdl.log; tail -3 gpurun_out/pytest_pdl.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for v in 0 1; do
  KRUL_PDL=$v timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_pdl$v.json 2> gpurun_out/bench_pdl$v.err
  python - <<PY
import json
b=json.load(open('gpurun_out/bench_pdl$v.json'))
r=b['rooflines']; h=b['roofline']
print('pdl=$v TTFT', b['ttft_p50_ms'], 'rc', b['config']['r_c'], 'h2d', b['restore']['h2d_ms'], h['class'], h['frac'], h['avg_launch_us'], 'ser', h['achieved_serialised'])
for k in ('attention','gemm','decode_expand','logits'):
    if k in r: print('  ', k, r[k]['frac'], r[k]['avg_launch_us'], r[k]['achieved_serialised'])
print('  calib', b['calibration']['calibration_ttft_ms'])
PY
done
