# main pass: next claim one ahead; claim sizes
timeout 900 python -m pytest tests -m gpu -x -q -k "render or pipelined or c1 or fused or sample_counts" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "FV_MAIN_CLAIM=2" "FV_MAIN_CLAIM=1" "FV_MAIN_CLAIM=4" "FV_MAIN_CLAIM=2"
