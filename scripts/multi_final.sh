#!/bin/bash
# Round-2 multi-GPU evidence on G GPUs of one box: replica bench (headline + per_model),
# table-wise sharded RMC2 bench, serving sweep (replicas, seed 11), sharding checks.
# usage: bash scripts/multi_final.sh G
G=${1:-2}
O=gpurun_out/r2_g$G
timeout 900 python -m pytest -m gpu -q -rs --timeout 800 -p no:cacheprovider tests/test_gpu_multi.py > $O.pytest_multi.log 2>&1
timeout 900 python bench.py --gpus $G > $O.bench.json 2> $O.bench.err
timeout 700 python bench.py --gpus $G --config rmc2 --shard table --step-batches 128 > $O.bench_rmc2_table.json 2> $O.bench_rmc2_table.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 \
  --master-port 29611 scripts/serving_sweep.py --modes synth --seeds 11 > $O.sweep.json 2> $O.sweep.err
