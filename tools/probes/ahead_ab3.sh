mkdir -p gpurun_out
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/ahead_ab3.log; }
for k in 2 4 6 8 3 5; do run a$k "FV_MARCH_AHEAD=$k"; done
run a4b "FV_MARCH_AHEAD=4"
