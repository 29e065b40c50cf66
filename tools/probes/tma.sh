mkdir -p gpurun_out
rm -f gpurun_out/tma_ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "conv3x3 or forward or end_to_end or pipelined or padded or strip" > gpurun_out/tma_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tma_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/tma_ab.log; }
run t1 ""; run t0 "FV_CONV_TMA=0"; run t1b ""; run t0b "FV_CONV_TMA=0"
