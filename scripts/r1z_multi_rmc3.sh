# RMC3 replicas at 2 and 4 GPUs (final build, Alg. 1 over d <= 4096)
mkdir -p gpurun_out
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29600+n)) bench.py --gpus $n --config rmc3 --no-cpu-baseline > gpurun_out/r1z_rmc3_${n}gpu.json 2> gpurun_out/r1z_rmc3_${n}gpu.err
  echo "n=$n rc=$?"
done
