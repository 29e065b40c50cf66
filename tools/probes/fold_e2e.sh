mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pipelined or graph or launch_variants or frames_to_host" > gpurun_out/folde2e_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/folde2e_tests.log
for m in 2 1 2 1; do echo "== split $m" >> gpurun_out/folde2e.log; FV_KCHAIN_SPLIT=$m timeout 300 python tools/probes/e2e_host.py >> gpurun_out/folde2e.log 2>&1; done
