# ray setup with 2 rays per thread (FV_SETUP_RPT=2) vs 1
for v in 1 2 1 2; do echo "== FV_SETUP_RPT=$v"; FV_SETUP_RPT=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/sr_spans.log > /dev/null; python tools/probes/launch_times.py gpurun_out/sr_spans.log 16 | sed -n 3,8p | awk '{printf "%s ", $3} END {print ""}'; done
timeout 600 python -m pytest tests -m gpu -x -q -k "launch_variants and SETUP_RPT" 2>&1 | tail -1
FV_SETUP_RPT=2 timeout 900 python -m pytest tests -m gpu -x -q -k "render or march or overflow or headline_e2e" 2>&1 | tail -1
