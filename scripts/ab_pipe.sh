# A/B: slot graphs vs S-D pipeline lanes (RMC1 unless $CFG), one box
B="--sla-queries 0 --no-cpu-baseline --e2e-steps 0 --roofline-steps 100 --sls-batches 100 --config ${CFG:-rmc1}"
P="import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['config']['items_per_s']/1e6,2), round(r['in_step_aggregate']['frac'],3), round(d['host_submit_us_per_step'],1))"
for i in 1 2; do
for a in "--streams 8" "--streams 8 --pipe 1" "--streams 8 --pipe 2" "--streams 16" "--streams 16 --pipe 2" "--streams 16 --pipe 4"; do
  echo -n "$a: "; timeout 300 python bench.py $B $a 2>/dev/null | python -c "$P"
done; done
