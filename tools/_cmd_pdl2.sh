for v in 0 1; do
  KRUL_PDL=$v timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_pdl$v.json 2> gpurun_out/bench_pdl$v.err
  echo "== KRUL_PDL=$v"; python tools/bench_brief.py gpurun_out/bench_pdl$v.json
done
