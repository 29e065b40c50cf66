# conv loader builds the decoder's 2x upsample (FV_UP_FUSE=1) vs a separate kernel
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "FV_UP_FUSE=0" "FV_UP_FUSE=1" "FV_UP_FUSE=0" "FV_UP_FUSE=1"
