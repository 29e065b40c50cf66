# fused K-stage logits: network parity tests, then A/B of FV_KFUSE on the C3 bench, then the timeline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forward or kernel_stage or end_to_end or pipelined or graph or launch_variants or strip or fused_pipeline" > gpurun_out/kfuse_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/kfuse_tests.log
timeout 900 python -m pytest tests/test_headline_parity.py -q -x -m gpu -k "network or end_to_end" > gpurun_out/kfuse_headline.log 2>&1
echo "headline rc=$?" >> gpurun_out/kfuse_headline.log
for k in 0 1 0 1; do
  echo "== kfuse $k" >> gpurun_out/kfuse_ab.log
  FV_KFUSE=$k timeout 600 python bench.py --no-cpu-baseline --no-sustained --steps 20 >> gpurun_out/kfuse_ab.log 2>&1
done
timeout 600 python tools/probes/timeline.py > gpurun_out/kfuse_timeline.log 2>&1
