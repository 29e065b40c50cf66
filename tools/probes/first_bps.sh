# first_list grid (blocks per SM)
for v in 2 8 4 2 8 4; do echo "== FV_FIRST_BPS=$v"; FV_FIRST_BPS=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/fb_spans.log > /dev/null; python tools/probes/launch_times.py gpurun_out/fb_spans.log 16 | sed -n 6,8p | awk '{printf "%s ", $3} END {print ""}'; done
FV_FIRST_BPS=8 timeout 600 python -m pytest tests -m gpu -x -q -k "launch_variants and COMP_HITS" 2>&1 | tail -1
