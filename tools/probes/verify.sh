# full GPU suite, the bench, the frame timeline
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -x -m gpu > gpurun_out/verify_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/verify_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/verify_bench.log 2>&1
timeout 600 python tools/probes/timeline.py > gpurun_out/verify_timeline.log 2>&1
