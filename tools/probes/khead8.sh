mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forward or kernel_stage or end_to_end or pipelined or graph" > gpurun_out/khead8_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/khead8_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/khead8_ab.log; }
run r8 ""
run r4 "FV_KHEAD_R=4"
run r8b ""
run r4b "FV_KHEAD_R=4"
