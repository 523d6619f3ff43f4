# round-1 evidence bundle on one GPU: full bench, ncu launch list, ncu --set full of the top kernels
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r1d_bench.json 2> gpurun_out/r1d_bench.err; echo bench_rc=$?
SHORT="--steps 40 --warmup 5 --sla-queries 0 --e2e-steps 0 --no-cpu-baseline --roofline-steps 10 --sls-batches 4"
timeout 600 python bench.py $SHORT > gpurun_out/r1d_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r1d.csv python bench.py $SHORT > gpurun_out/r1d_ncu_list.log 2>&1; echo list_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sls_synth|k_mlp_chain|k_interact|k_gen_dense_seg" --launch-skip 40 -c 8 -o gpurun_out/prof_r1d -f python bench.py $SHORT > gpurun_out/r1d_ncu_full.log 2>&1; echo full_rc=$?
timeout 300 python scripts/sls_probe.py --synth 1024 --iters 20 > gpurun_out/r1d_probe.log 2>&1; echo probe_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:k_sls_synth -c 3 -o gpurun_out/prof_r1d_sls1024 -f python scripts/sls_probe.py --synth 1024 --iters 20 > gpurun_out/r1d_ncu_sls.log 2>&1; echo sls_rc=$?
