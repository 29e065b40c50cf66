mkdir -p gpurun_out
rm -f gpurun_out/dxn_ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "forward or end_to_end or pipelined or launch_variants or padded" > gpurun_out/dxn_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/dxn_tests.log
timeout 900 python -m pytest tests/test_headline_parity.py -q -m gpu -k "network or end_to_end" >> gpurun_out/dxn_tests.log 2>&1
echo "headline rc=$?" >> gpurun_out/dxn_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/dxn_ab.log; }
run d1 ""; run d0 "FV_KHEAD_DXN=0"; run d1b ""; run d0b "FV_KHEAD_DXN=0"
