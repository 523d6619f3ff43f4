# A/B of library variants (REC_LIB_PATH) on one box: RMC1 step throughput + SLS rooflines
B="--sla-queries 0 --no-cpu-baseline --e2e-steps 0 --roofline-steps 100 --sls-batches 200 --mlp-batch 0 --config ${CFG:-rmc1}"
P="import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=lambda k: round(r.get(k,{}).get('frac',-1),3); print(round(d['value']), round(r['frac'],3), g('serialized'), g('isolated'), g('in_step_aggregate'))"
for i in 1 2; do
for L in default "$@"; do
  echo -n "$L "
  if [ "$L" = default ]; then timeout 300 python bench.py $B 2>/dev/null | python -c "$P"
  else REC_LIB_PATH=$PWD/$L timeout 300 python bench.py $B 2>/dev/null | python -c "$P"; fi
done; done
