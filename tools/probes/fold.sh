mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "pipelined or graph or launch_variants or frames_to_host or strip or end_to_end" > gpurun_out/fold_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fold_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/fold_tests.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fold_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/fold_ab.log; }
run f2a1 ""
run f1 "FV_KCHAIN_SPLIT=1"
run f2a2 "FV_KCHAIN_AT=2"
run f2a3 "FV_KCHAIN_AT=3"
run f2a1b ""
run f1b "FV_KCHAIN_SPLIT=1"
