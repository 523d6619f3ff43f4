#!/bin/bash
# A/B of co-location depth and GEMM tiling for a dense-heavy workload (saturation QPS only).
# usage: bash scripts/ab_dense.sh <config> <out-prefix>
CFG=${1:-rmc3}
OUT=${2:-gpurun_out/ab_dense}
Q="--config $CFG --per-model '' --sla-queries 0 --mlp-batch 0 --e2e-steps 0 --no-cpu-baseline --steps 10 --step-batches 256"
run() {  # tag, env, args
  local tag=$1; shift
  local envs=$1; shift
  env $envs timeout 300 python bench.py --config $CFG --per-model "" --sla-queries 0 --mlp-batch 0 \
    --e2e-steps 0 --no-cpu-baseline --steps 10 --step-batches 256 "$@" > $OUT.$tag.json 2> $OUT.$tag.err
  python -c "import json;d=json.loads(open('$OUT.$tag.json').read().strip().splitlines()[-1]);print('$tag', round(d['value']), d['roofline']['in_step_aggregate']['frac'], d['mlp']['in_step_aggregate']['frac'], d['breakdown_us_per_batch_single_stream'])"
}
run s16 "X=1" --streams 16
run s32 "X=1" --streams 32
run s48 "X=1" --streams 48
run s16_narrow64 "REC_GEMM_NARROW=64" --streams 16
run s32_narrow64 "REC_GEMM_NARROW=64" --streams 32
run s16_narrow148 "REC_GEMM_NARROW=148" --streams 16
