# dynamic conv tile claims (one ahead): conv tests, then bench with marcher claim sizes
timeout 600 python -m pytest tests -m gpu -x -q -k "conv or forward or pipelined or kernel_timing" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "FV_MAIN_CLAIM=32" "FV_MAIN_CLAIM=4" "FV_MAIN_CLAIM=32" "FV_MAIN_CLAIM=4"
