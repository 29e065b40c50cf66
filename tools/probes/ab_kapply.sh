# K-stage apply passes: pixel pairs with 8-byte loads vs per pixel (FV_KAPPLY_V=1); parity first
timeout 900 python -m pytest tests -m gpu -x -q -k "forward or kernel_stage or end_to_end or pipelined or graph or fused or frames" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "FV_KAPPLY_V=1" "FV_KAPPLY_V=2" "FV_KAPPLY_V=1" "FV_KAPPLY_V=2"
