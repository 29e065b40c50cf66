mkdir -p gpurun_out
FV_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c5 --shard --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/shard2.log 2>&1
echo "rc=$?" >> gpurun_out/shard2.log
