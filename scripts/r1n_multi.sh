#!/bin/bash
# Multi-GPU refresh (2 and 4 GPUs, replicas, default bench) with the current build.
set -u
mkdir -p gpurun_out
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500+n)) bench.py --gpus $n > gpurun_out/r1n_bench_${n}gpu.json 2> gpurun_out/r1n_bench_${n}gpu.err
  echo "n=$n rc=$?"
  tail -c 1500 gpurun_out/r1n_bench_${n}gpu.json
done
