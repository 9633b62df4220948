# The other BASELINE.json configs through bench.py (same kernels), round-2 evidence run.
mkdir -p gpurun_out
timeout 900 python bench.py --config tiny-512 --steps 20 --warmup 3 > gpurun_out/bench_tiny.json 2> gpurun_out/bench_tiny.err; echo "tiny exit $?"; tail -2 gpurun_out/bench_tiny.err
timeout 900 python bench.py --config mistral-7b-32k --steps 10 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_mistral.json 2> gpurun_out/bench_mistral.err; echo "mistral exit $?"; tail -2 gpurun_out/bench_mistral.err
timeout 1500 python bench.py --config llama3-70b-16k --steps 5 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_70b.json 2> gpurun_out/bench_70b.err; echo "70b exit $?"; tail -2 gpurun_out/bench_70b.err
timeout 2400 python bench.py --config llama3-8b-batch256 --no-cpu-baseline --no-policies > gpurun_out/bench_batch256.json 2> gpurun_out/bench_batch256.err; echo "batch exit $?"; tail -2 gpurun_out/bench_batch256.err
for f in tiny mistral 70b batch256; do echo "== $f"; python tools/bench_brief.py gpurun_out/bench_$f.json | head -8; done
