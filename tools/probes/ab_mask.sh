# mask kernel: warp-wide look-back window
timeout 900 python -m pytest tests -m gpu -x -q -k "mask or scatter or render_sparse or c1 or pipelined or fused" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "X=1" "X=2"
