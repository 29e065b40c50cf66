# shadow pass: second trilinear plane through the LSU path (FV_SHADOW_MIX=1) vs both planes from the texture
python -m pytest tests -m gpu -x -q -k "render or sample_counts or pipelined or end_to_end or c1" > gpurun_out/t_render.log 2>&1; tail -2 gpurun_out/t_render.log
FV_SHADOW_MIX=1 python -m pytest tests -m gpu -x -q -k "render or sample_counts or c1" > gpurun_out/t_render_mix.log 2>&1; tail -2 gpurun_out/t_render_mix.log
bash tools/probes/ab_env.sh "FV_SHADOW_MIX=0" "FV_SHADOW_MIX=1" "FV_SHADOW_MIX=0" "FV_SHADOW_MIX=1"
