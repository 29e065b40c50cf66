# upsample with RP input rows per thread (FV_UP_ROWS=1/2/4): per-launch times, bit-identity
for v in 1 2 4 1 2 4; do echo "== FV_UP_ROWS=$v"; FV_UP_ROWS=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/up_spans_$v.log | grep -i "netops"; python tools/probes/launch_times.py gpurun_out/up_spans_$v.log 16 | grep -i "netops" | head -3; done
timeout 900 python -m pytest tests -m gpu -x -q -k "launch_variants and (UP_ROWS or N80)" 2>&1 | tail -2
