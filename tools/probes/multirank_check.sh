# Functional check of bench.py's torchrun paths on a 1-GPU box: 2 ranks share cuda:0 and time
# through gloo (FV_DIST_BACKEND=gloo). The numbers are meaningless (the ranks contend for one GPU);
# the check is that every path runs, rank 0 alone prints one JSON line and the other ranks exit 0.
run() {
  FV_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 "$@"
}
echo "== independent streams";   run --steps 5 --warmup 3 --no-cpu-baseline | tail -1 | cut -c1-300
echo "== sharded c5";            run --config c5 --shard --steps 3 --warmup 3 --no-cpu-baseline | tail -1 | cut -c1-300
echo "== reference arm";         run --impl reference --steps 1 --warmup 0 | tail -1 | cut -c1-300
