# pair conv with TMA tensor-map hand-off (FV_CONV_PAIR=1, FV_PAIR_TMA default) -- correctness first, under timeouts
FV_CONV_PAIR=1 timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "conv3x3" 2>&1 | tail -3
FV_CONV_PAIR=1 timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "forward or end_to_end or pipelined" 2>&1 | tail -3
for v in "0 1" "1 1" "1 0" "0 1" "1 1"; do set -- $v; echo "== FV_CONV_PAIR=$1 FV_PAIR_TMA=$2"; FV_CONV_PAIR=$1 FV_PAIR_TMA=$2 FV_KTIME_LOG=1 timeout 300 python tools/probes/kernel_times.py 3 8 2> gpurun_out/pt_spans.log | grep conv; python tools/probes/launch_times.py gpurun_out/pt_spans.log 8 | grep conv | head -16 | awk '{printf "%s ", $3} END {print ""}'; done
