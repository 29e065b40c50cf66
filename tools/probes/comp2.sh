mkdir -p gpurun_out
rm -f gpurun_out/comp2_ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "render or pipelined or end_to_end or overflow or frames_to_host" > gpurun_out/comp2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/comp2_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/comp2_ab.log; }
run n ""; run o "FV_LIBFOVNET=ab_tmp/lib_old.so"; run n2 ""; run o2 "FV_LIBFOVNET=ab_tmp/lib_old.so"
