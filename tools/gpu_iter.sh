#!/bin/bash
# One GPU iteration: bash tools/gpu_iter.sh TAG "pytest -k expr" "ncu kernel regex" [bench args]
TAG=$1; KEXPR=$2; NCU_RE=$3; shift 3
OUT=gpurun_out; mkdir -p $OUT
if [ -n "$KEXPR" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_$TAG.log
  tail -3 $OUT/pytest_$TAG.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
tail -2 $OUT/smoke_$TAG.log
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline "$@" > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
tail -1 $OUT/bench_$TAG.err
python - <<PY
import json
try:
    b=json.load(open('$OUT/bench_$TAG.json'))
    print('TTFT', b['ttft_p50_ms'], 'e2e', b['e2e']['ttft_p50_ms'], 'rc', b['config']['r_c'], 'restore', b['restore'])
    print('roofline', b['roofline']['class'], b['roofline']['frac'], b['roofline']['avg_launch_us'])
    for k,v in b['rooflines'].items(): print(' ', k, v.get('frac'), v.get('avg_launch_us'), v.get('ms_per_step'), v.get('achieved_serialised'))
    print('policies', {k:v['ttft_ms'] for k,v in b.get('policies',{}).items()})
    print('calib', b['calibration'].get('calibration_ttft_ms'))
except Exception as e: print('bench parse failed', e)
PY
if [ -n "$NCU_RE" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"$NCU_RE" -s 5 -c 1 -o $OUT/prof_$TAG -f python tools/profile_step.py > $OUT/prof_$TAG.log 2>&1
  tail -1 $OUT/prof_$TAG.log
fi
