#!/bin/bash
# A/B of co-location depth and GEMM tiling for a dense-heavy workload (saturation QPS only).
# usage: bash scripts/ab_dense.sh <config> <out-prefix> tag:ENV=V:streams ...   (ENV X=1 = none)
CFG=${1:-rmc3}; shift
OUT=${1:-gpurun_out/ab_dense}; shift
run() {  # tag, env, args
  local tag=$1; shift
  local envs=$1; shift
  env $envs timeout 300 python bench.py --config $CFG --per-model "" --sla-queries 0 --mlp-batch 0 \
    --e2e-steps 0 --no-cpu-baseline --steps 10 --step-batches 256 "$@" > $OUT.$tag.json 2> $OUT.$tag.err
  python -c "import json;d=json.loads(open('$OUT.$tag.json').read().strip().splitlines()[-1]);print('$tag', round(d['value']), d['roofline']['in_step_aggregate']['frac'], d['mlp']['in_step_aggregate']['frac'], d['breakdown_us_per_batch_single_stream'])"
}
for spec in "$@"; do  # tag:ENV=V:streams
  IFS=: read tag envs streams <<< "$spec"
  run $tag "$envs" --streams $streams
done
