# ray headers at hit-list positions, composite over the hits only (FV_COMP_HITS=1) x main-pass block (FV_MAIN_U)
for v in "0 2" "1 2" "1 1" "0 2" "1 2" "1 1"; do set -- $v; echo "== FV_COMP_HITS=$1 FV_MAIN_U=$2"; FV_COMP_HITS=$1 FV_MAIN_U=$2 FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/ch2_spans.log | grep -i "march"; python tools/probes/launch_times.py gpurun_out/ch2_spans.log 16 | sed -n 3,8p; done
timeout 900 python -m pytest tests -m gpu -x -q -k "launch_variants and (COMP_HITS or MAIN_U)" 2>&1 | tail -1
FV_COMP_HITS=1 timeout 900 python -m pytest tests -m gpu -x -q -k "render or march or headline_e2e or overflow or shard or viewer" 2>&1 | tail -1
