# D.head TAPN + strip upsample: network / pipeline tests, then timeline A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forward or kernel_stage or end_to_end or pipelined or graph or launch_variants or strip or fused_pipeline or conv3x3" > gpurun_out/khead_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/khead_tests.log
timeout 900 python -m pytest tests/test_headline_parity.py -q -x -m gpu -k "network or end_to_end" > gpurun_out/khead_headline.log 2>&1
echo "headline rc=$?" >> gpurun_out/khead_headline.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/khead_ab.log; }
run new ""
run tapn0 "FV_KHEAD_TAPN=0"
run up1 "FV_UPSAMPLE_V=1"
run new2 ""
run old "FV_KHEAD_TAPN=0 FV_UPSAMPLE_V=1"
