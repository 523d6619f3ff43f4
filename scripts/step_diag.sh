#!/bin/bash
# diagnostic (needs the -DREC_DEBUG_KNOBS library, e.g. variants/libhercules_rec_diag.so):
# step throughput with stages dropped (REC_STEP_DIAG bits: 1 bottom, 2 interaction+top,
# 4 interaction alone) -> the marginal cost of each dense stage in the co-located step.
# usage: REC_LIB_PATH=$PWD/variants/libhercules_rec_diag.so bash scripts/step_diag.sh rmc3 32
CFG=${1:-rmc3}; ST=${2:-32}
for v in 0 1 2 4 3; do
  REC_STEP_DIAG=$v timeout 300 python bench.py --config $CFG --streams $ST --per-model "" --sla-queries 0 \
    --mlp-batch 0 --e2e-steps 0 --no-cpu-baseline --caller-batches 0 --steps 10 --step-batches 256 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG streams=$ST diag=$v', round(d['value']), round(d['roofline']['in_step_aggregate']['frac'],3))"
done
