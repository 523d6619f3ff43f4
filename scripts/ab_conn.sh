#!/bin/bash
# A/B: CUDA_DEVICE_MAX_CONNECTIONS (hardware work queues shared by the co-located streams).
# usage: bash scripts/ab_conn.sh <out-prefix>
OUT=${1:-gpurun_out/ab_conn}
for cfg in rmc1 rmc3; do
  for c in 8 16 32; do
    CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python bench.py --config $cfg --per-model "" --sla-queries 0 \
      --mlp-batch 0 --e2e-steps 0 --no-cpu-baseline --caller-batches 0 --steps 10 --step-batches 256 \
      > $OUT.$cfg.c$c.json 2> $OUT.$cfg.c$c.err
    python -c "import json;d=json.loads(open('$OUT.$cfg.c$c.json').read().strip().splitlines()[-1]);print('$cfg conn=$c', round(d['value']), round(d['roofline']['in_step_aggregate']['frac'],3), d['config']['streams_per_gpu'])"
  done
done
