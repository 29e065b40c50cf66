# main pass with 32 samples per warp block (FV_MAIN_U=1) vs 64: per-launch march times, bit-identity of frames is NOT expected (same samples, same order)
for v in 2 1 2 1; do echo "== FV_MAIN_U=$v"; FV_MAIN_U=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/mu_spans_$v.log | grep -i "march\|frames"; python tools/probes/launch_times.py gpurun_out/mu_spans_$v.log 16 | sed -n 3,5p; done
for v in 2 1; do FV_MAIN_U=$v timeout 900 python -m pytest tests -m gpu -x -q -k "render or march or headline_e2e or overflow" 2>&1 | tail -1; done
