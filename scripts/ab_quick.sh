# quick RMC1/RMC3 step throughput at 8 and 16 streams (one box)
P="import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['config']['items_per_s']/1e6,2), round(r['in_step_aggregate']['frac'],3), d['breakdown_us_per_batch_single_stream'])"
for c in ${CFGS:-rmc1 rmc3}; do for st in 8 16; do
  echo -n "$c streams=$st: "; timeout 300 python bench.py --config $c --streams $st --sla-queries 0 --no-cpu-baseline --e2e-steps 0 --roofline-steps 100 --sls-batches 100 2>/dev/null | python -c "$P"
done; done
