# diagnostic: step throughput with stages dropped (REC_STEP_DIAG bits: 1 bottom, 2 interaction+top)
B="--sla-queries 0 --no-cpu-baseline --e2e-steps 0 --roofline-steps 100 --sls-batches 100 --mlp-batch 0"
P="import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['config']['items_per_s']/1e6,2), round(d['roofline']['in_step_aggregate']['frac'],3))"
for cfg in "${@:-rmc1}"; do for st in 8 16 32; do
for v in 0 1 2 3; do echo -n "$cfg streams=$st diag=$v "; REC_STEP_DIAG=$v timeout 300 python bench.py --config $cfg --streams $st $B 2>/dev/null | python -c "$P"; done
done; done
