# A/B of bench.py argument sets on one box (RMC1 step throughput; args: "--opt v" ...)
B="--sla-queries 0 --no-cpu-baseline --e2e-steps 0 --roofline-steps 100 --sls-batches 100 --mlp-batch 0 --config ${CFG:-rmc1}"
P="import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['config']['items_per_s']/1e6,2), round(d['roofline']['in_step_aggregate']['frac'],3))"
for i in 1 2; do for a in "" "$@"; do
  echo -n "[$a]: "; timeout 300 python bench.py $B $a 2>/dev/null | python -c "$P"
done; done
