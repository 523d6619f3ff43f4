# A/B on one box: build/prev (older commit worktree) vs current-tree variants, alternating
B="--sla-queries 0 --no-cpu-baseline --e2e-steps 0 --roofline-steps 100"
P="import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['breakdown_us_per_batch_single_stream']['sls'],2), round(d['roofline']['frac'],3) if 'roofline' in d else '')"
for i in 1 2; do
echo -n "prev    "; (cd build/prev && timeout 300 python bench.py $B 2>/dev/null | python -c "$P")
echo -n "cur     "; timeout 300 python bench.py $B --sls-batches 8 2>/dev/null | python -c "$P"
echo -n "pdl0    "; REC_PDL=0 timeout 300 python bench.py $B --sls-batches 8 2>/dev/null | python -c "$P"
done
