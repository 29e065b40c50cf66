mkdir -p gpurun_out
FV_CONV_R8=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forward or conv3x3 or end_to_end or pipelined" > gpurun_out/r8_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r8_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/r8_ab.log; }
run c8 "FV_CONV_R8=1"
run c4 ""
run c8b "FV_CONV_R8=1"
run c4b ""
