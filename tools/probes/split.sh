mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "pipelined or graph or launch_variants or frames_to_host or strip or fused_pipeline or end_to_end" > gpurun_out/split_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/split_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/split_tests.log 2>&1
echo "smoke rc=$?" >> gpurun_out/split_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/split_ab.log; }
run s1 ""
run s0 "FV_KCHAIN_SPLIT=0"
run s1b ""
run s0b "FV_KCHAIN_SPLIT=0"
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/split_bench.log 2>&1
