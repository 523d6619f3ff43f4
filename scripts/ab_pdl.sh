for i in 1 2; do
for v in 1 0; do
REC_PDL=$v timeout 300 python bench.py --sla-queries 0 --no-cpu-baseline --e2e-steps 0 --roofline-steps 100 --sls-batches 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=$v', round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['in_step_aggregate']['frac'],3), d['clocks']['sm_mhz'])"
done; done
