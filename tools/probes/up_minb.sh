# upsample rows kernel register bound (FV_UP_MINB=1 / 8)
for v in 1 8 1 8; do echo "== FV_UP_MINB=$v"; FV_UP_MINB=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/um_spans.log > /dev/null; python tools/probes/launch_times.py gpurun_out/um_spans.log 16 | grep netops | head -3 | awk '{printf "%s ", $3} END {print ""}'; done
FV_UP_MINB=8 timeout 600 python -m pytest tests -m gpu -x -q -k "launch_variants and UP_ROWS" 2>&1 | tail -1
