# composite: warp per ray, no chunk_fill read; grid size
timeout 600 python -m pytest tests -m gpu -x -q -k "render or pipelined or c1 or fused or shard or frames" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "FV_COMP_BLOCKS=16" "FV_COMP_BLOCKS=32" "FV_COMP_BLOCKS=16"
