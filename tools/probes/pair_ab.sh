mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "conv3x3 or forward" > gpurun_out/pair_tests2.log 2>&1
for v in 0 1; do
  FV_CONV_PAIR=$v FV_KTIME_LOG=1 timeout 300 python tools/probes/kernel_times.py 10 6 > /dev/null 2> gpurun_out/pair_spans_$v.log
  python tools/probes/launch_times.py gpurun_out/pair_spans_$v.log 6 > gpurun_out/pair_launch_$v.txt
done
make -s -C paper_2209_09965_b200/csrc clean
make -s -C paper_2209_09965_b200/csrc -j16 EXTRA=-DFV_CONV_PROFILE=1 > gpurun_out/build_prof.log 2>&1
FV_CONV_PAIR=1 FV_CONV_PROF=1 FV_GRAPH=0 timeout 600 python tools/profile_frame.py c3 3 > gpurun_out/pair_waits2.log 2>&1
