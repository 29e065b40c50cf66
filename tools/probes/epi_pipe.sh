# plain conv epilogue with the next item's TMEM loads in flight (FV_EPI_PIPE=1) vs one item at a time
for v in 0 1 0 1; do echo "== FV_EPI_PIPE=$v"; FV_EPI_PIPE=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/ep_spans.log | grep conv; python tools/probes/launch_times.py gpurun_out/ep_spans.log 16 | grep conv | head -16 | awk '{printf "%s ", $3} END {print ""}'; done
for v in 0 1; do FV_EPI_PIPE=$v timeout 900 python -m pytest tests -m gpu -x -q -k "conv or forward or headline_network" 2>&1 | tail -1; done
