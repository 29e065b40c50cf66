mkdir -p gpurun_out
rm -f gpurun_out/lin_ab.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/lin_ab.log; }
run d "" ; run a412 "FV_SHADOW_LIN=4,12"; run a808 "FV_SHADOW_LIN=8,8"; run a416 "FV_SHADOW_LIN=4,16"; run a610 "FV_SHADOW_LIN=6,10"; run d2 ""
