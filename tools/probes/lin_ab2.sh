mkdir -p gpurun_out
rm -f gpurun_out/lin_ab2.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/lin_ab2.log; }
for i in 1 2 3; do run d$i ""; run s$i "FV_SHADOW_LIN=6,10"; done
