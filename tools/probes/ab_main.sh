# main-pass lookahead block (C3 bench A/B) + parity subset
python -m pytest tests -m gpu -x -q -k "render or sample_counts or pipelined or end_to_end or c1 or shard or fused" > gpurun_out/t_render.log 2>&1; tail -3 gpurun_out/t_render.log
bash tools/probes/ab_env.sh "FV_MAIN_LA=0" "FV_MAIN_LA=1" "FV_MAIN_MINB=4" "FV_MAIN_MINB=6"
