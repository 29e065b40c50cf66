# mask with incremental noise / pixel coordinates: bit-exact mask tests, per-launch times
timeout 900 python -m pytest tests -m gpu -x -q -k "mask and not headline" 2>&1 | tail -1
FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/mi_spans.log | grep -i "mask"; python tools/probes/launch_times.py gpurun_out/mi_spans.log 16 | sed -n 1,2p
