# The other BASELINE.json configs through bench.py (same kernels).
mkdir -p gpurun_out
timeout 900 python bench.py --config mistral-7b-32k --steps 5 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_mistral.json 2> gpurun_out/bench_mistral.err; echo "mistral exit $?"; tail -3 gpurun_out/bench_mistral.err
timeout 1200 python bench.py --config llama3-70b-16k --steps 5 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_70b.json 2> gpurun_out/bench_70b.err; echo "70b exit $?"; tail -3 gpurun_out/bench_70b.err
timeout 900 python bench.py --config llama3-8b-batch256 --convs 6 --steps 6 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; echo "batch exit $?"; tail -3 gpurun_out/bench_batch.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
