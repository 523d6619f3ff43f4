# final round-1 evidence on one GPU: plain short run, ncu launch list, ncu --set full of the
# SLS / fused-MLP / interaction kernels (same short command; never under torchrun)
mkdir -p gpurun_out
SHORT="--steps 64 --warmup 16 --sla-queries 0 --e2e-steps 0 --no-cpu-baseline --roofline-steps 10 --sls-batches 4 --mlp-batch 0"
timeout 600 python bench.py $SHORT > gpurun_out/r1z_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_r1z.csv python bench.py $SHORT > gpurun_out/r1z_ncu_list.log 2>&1; echo list_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sls_synth|k_mlp_chain|k_interact|k_gen_dense_seg" --launch-skip 60 -c 8 -o gpurun_out/prof_r1z -f python bench.py $SHORT > gpurun_out/r1z_ncu_full.log 2>&1; echo full_rc=$?
