mkdir -p gpurun_out
rm -f gpurun_out/minb_ab.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/minb_ab.log; }
run m6 ""; run m8 "FV_MAIN_MINB_RT=8"; run m10 "FV_MAIN_MINB_RT=10"; run m6b ""; run m8b "FV_MAIN_MINB_RT=8"
