# render-branch carveout / occupancy A/B on the frame timeline
mkdir -p gpurun_out
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/carve_ab.log; }
run base ""
run c100 "FV_MARCH_CARVEOUT=100"
run c100o50 "FV_MARCH_CARVEOUT=100 FV_MARCH_OCC=50"
run o50 "FV_MARCH_OCC=50"
run c100o35 "FV_MARCH_CARVEOUT=100 FV_MARCH_OCC=35"
run base2 ""
run c50 "FV_MARCH_CARVEOUT=50"
run kf0 "FV_KFUSE=0"
