mkdir -p gpurun_out
rm -f gpurun_out/refill_ab.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/refill_ab.log; }
run d ""; run r4 "FV_SHADOW_REFILL=4"; run r12 "FV_SHADOW_REFILL=12"; run r16 "FV_SHADOW_REFILL=16"; run c32 "FV_SHADOW_CLAIM=32"; run c128 "FV_SHADOW_CLAIM=128"; run d2 ""
