mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "conv3x3" > gpurun_out/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "forward or end_to_end or pipelined or strip" >> gpurun_out/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_tests.log
FV_KTIME_LOG=1 timeout 300 python tools/probes/kernel_times.py 10 6 > gpurun_out/pair_times.log 2> gpurun_out/pair_spans.log
python tools/probes/launch_times.py gpurun_out/pair_spans.log 6 > gpurun_out/pair_launch.txt
