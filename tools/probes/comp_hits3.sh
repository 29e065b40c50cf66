# composite with the next header prefetched (default now: hit-indexed headers, 32-sample main blocks); C3 / C2 / C5 main-pass block A/B
for v in 0 1; do echo "== C3 FV_COMP_HITS=$v"; FV_COMP_HITS=$v FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/ch3_spans.log | grep -i "march_comp"; python tools/probes/launch_times.py gpurun_out/ch3_spans.log 16 | sed -n 6,8p; done
for c in c2 c5; do for u in 2 1; do echo "== $c FV_MAIN_U=$u"; FV_MAIN_U=$u python tools/probes/kernel_times.py 3 8 $c | grep -i "march\|frames"; done; done
timeout 900 python -m pytest tests -m gpu -x -q -k "launch_variants and (COMP_HITS or MAIN_U)" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "render or march or headline_e2e or overflow or viewer or pipelined" 2>&1 | tail -1
