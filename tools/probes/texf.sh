mkdir -p gpurun_out
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/texf_ab.log; }
run f1 ""
run f2 "FV_TEX_FILTER=2"
run f1b ""
run f2b "FV_TEX_FILTER=2"
