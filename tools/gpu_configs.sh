mkdir -p gpurun_out
timeout 900 python bench.py --config mistral-7b-32k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mistral.json 2> gpurun_out/bench_mistral.err; echo "mistral exit $?"; tail -3 gpurun_out/bench_mistral.err
timeout 1200 python bench.py --config llama3-70b-16k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_70b.json 2> gpurun_out/bench_70b.err; echo "70b exit $?"; tail -3 gpurun_out/bench_70b.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
