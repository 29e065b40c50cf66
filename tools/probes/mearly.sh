mkdir -p gpurun_out
rm -f gpurun_out/mearly_ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pipelined or graph or launch_variants or frames_to_host" > gpurun_out/mearly_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mearly_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/mearly_ab.log; }
run e1 ""; run e0 "FV_MASK_EARLY=0"; run e1b ""; run e0b "FV_MASK_EARLY=0"
