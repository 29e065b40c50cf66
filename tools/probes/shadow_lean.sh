mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "render or sample_counts or overflow or end_to_end or pipelined" > gpurun_out/lean_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/lean_tests.log
timeout 1200 python -m pytest tests/test_headline_parity.py -q -m gpu -k "march or end_to_end" >> gpurun_out/lean_tests.log 2>&1
echo "headline rc=$?" >> gpurun_out/lean_tests.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/lean_ab.log; }
run l1 ""
run l1b ""
