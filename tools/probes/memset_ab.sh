mkdir -p gpurun_out
rm -f gpurun_out/memset_ab.log
run() { env $2 TL_TAG=_$1 timeout 300 python tools/probes/timeline.py 2>/dev/null | tail -1 >> gpurun_out/memset_ab.log; }
run k "" ; run m "FV_ZERO_MEMSET=1"; run k2 ""; run m2 "FV_ZERO_MEMSET=1"
timeout 300 python tools/probes/e2e_host.py > gpurun_out/memset_e2e_k.log 2>&1
FV_ZERO_MEMSET=1 timeout 300 python tools/probes/e2e_host.py > gpurun_out/memset_e2e_m.log 2>&1
