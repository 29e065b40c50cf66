# 64-column conv pipeline depth: resident-weight 5 -> 6 stages, streamed 4 -> 5 (FV_N64_S=6 / 5)
for v in 0 6 5 0 6 5; do echo "== FV_N64_S=$v"; FV_N64_S=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/ns_spans.log | grep conv; python tools/probes/launch_times.py gpurun_out/ns_spans.log 16 | grep conv | head -16 | awk '{printf "%s ", $3} END {print ""}'; done
