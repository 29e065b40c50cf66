mkdir -p gpurun_out
rm -f gpurun_out/rev_ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "forward or pipelined or launch_variants" > gpurun_out/rev_tests.log 2>&1
echo "rc=$?" >> gpurun_out/rev_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/rev_ab.log; }
for i in 1 2 3; do run r$i ""; run f$i "FV_CONV_REV=0"; done
