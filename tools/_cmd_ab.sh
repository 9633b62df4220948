# A/B of an env knob on the short bench: bash tools/_cmd_ab.sh VAR "v1 v2"
VAR=$1; VALS=$2
for v in $VALS; do
  env $VAR=$v timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_ab_$v.json 2> gpurun_out/bench_ab_$v.err
  echo "== $VAR=$v"; python tools/bench_brief.py gpurun_out/bench_ab_$v.json | grep -v "None None None"
done
