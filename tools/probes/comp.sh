mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "render or sample_counts or overflow or end_to_end or pipelined or graph or frames_to_host or launch_variants or mask" > gpurun_out/comp_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/comp_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/comp_ab.log; }
run c1 ""
run c1b ""
timeout 300 python tools/probes/e2e_host.py > gpurun_out/comp_e2e.log 2>&1
timeout 300 python tools/probes/timeline_e2e.py >> gpurun_out/comp_e2e.log 2>&1
