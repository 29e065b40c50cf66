mkdir -p gpurun_out
for v in 0 1; do
  FV_K0_TAPN=$v FV_KTIME_LOG=1 timeout 600 python tools/probes/kernel_times.py 10 8 > gpurun_out/k0_times_$v.log 2> gpurun_out/k0_spans_$v.log
  python tools/probes/launch_times.py gpurun_out/k0_spans_$v.log 8 > gpurun_out/k0_launch_$v.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "forward or end_to_end" > gpurun_out/k0_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k0_tests.log
