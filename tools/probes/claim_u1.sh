# main-pass ray claims per atomic with 32-sample blocks
for c in 2 1 4 8 2 1 4 8; do echo "== FV_MAIN_CLAIM=$c"; FV_MAIN_CLAIM=$c FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/cl_spans.log >/dev/null; python tools/probes/launch_times.py gpurun_out/cl_spans.log 16 | sed -n 4,4p; done
