mkdir -p gpurun_out
rm -f gpurun_out/pred_ab.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/pred_ab.log; }
run p1 ""; run p0 "FV_LIBFOVNET=ab_tmp/lib_pred0.so"; run p1b ""; run p0b "FV_LIBFOVNET=ab_tmp/lib_pred0.so"
