#!/bin/bash
# batch config on 1 GPU (few conversations) + a 2-rank torchrun with both ranks on GPU 0 (gloo)
mkdir -p gpurun_out
timeout 900 python bench.py --config llama3-8b-batch256 --convs 6 > gpurun_out/bench_batch1.json 2> gpurun_out/bench_batch1.err; echo "batch exit $?"; tail -2 gpurun_out/bench_batch1.err
KRUL_BENCH_DEVICE=0 KRUL_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "2rank exit $?"; tail -3 gpurun_out/bench_2rank.err
KRUL_BENCH_DEVICE=0 KRUL_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_2rank_ref.json 2> gpurun_out/bench_2rank_ref.err; echo "2rank ref exit $?"
