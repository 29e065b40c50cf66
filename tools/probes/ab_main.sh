# main pass with claims two ahead + cp.async list entries; chunk pool sizes; graph replay test
timeout 900 python -m pytest tests -m gpu -x -q -k "render or pipelined or c1 or fused or shard or frames or graph or sample_counts" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_env.sh "FV_CHUNK_POOL=8" "FV_CHUNK_POOL=16" "FV_CHUNK_POOL=32" "FV_MAIN_CLAIM=4" "FV_CHUNK_POOL=8"
