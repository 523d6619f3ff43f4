# evidence bundle on one GPU: full bench (RMC1), RMC2/RMC3 lines, ncu launch list + --set full
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r1j_bench.json 2> gpurun_out/r1j_bench.err; echo bench_rc=$?
for c in rmc2 rmc3 mtwnd; do timeout 700 python bench.py --config $c --no-cpu-baseline > gpurun_out/r1j_bench_$c.json 2> gpurun_out/r1j_bench_$c.err; echo ${c}_rc=$?; done
SHORT="--steps 64 --warmup 16 --sla-queries 0 --e2e-steps 0 --no-cpu-baseline --roofline-steps 10 --sls-batches 4 --mlp-batch 0"
timeout 600 python bench.py $SHORT > gpurun_out/r1j_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_r1j.csv python bench.py $SHORT > gpurun_out/r1j_ncu_list.log 2>&1; echo list_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sls_synth|k_mlp_chain|k_interact|k_gen_dense_seg" --launch-skip 60 -c 8 -o gpurun_out/prof_r1j -f python bench.py $SHORT > gpurun_out/r1j_ncu_full.log 2>&1; echo full_rc=$?
