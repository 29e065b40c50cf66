# reconstruct() as captured CUDA graphs vs eager launches
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "FV_GRAPH=0" "FV_GRAPH=1" "FV_GRAPH=0" "FV_GRAPH=1"
