mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "forward or kernel_stage or end_to_end or pipelined or graph_replay" > gpurun_out/k0_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k0_tests.log
FV_PARITY_REPORT=gpurun_out/hp_k0.json timeout 900 python -m pytest tests/test_headline_parity.py -q -k "C3 and network" > gpurun_out/k0_headline.log 2>&1; echo "rc=$?" >> gpurun_out/k0_headline.log
for v in "FV_K0_TAPN=1" "FV_K0_TAPN=0" "FV_K0_TAPN=1"; do
  echo "== $v" >> gpurun_out/k0_ab.log
  env $v timeout 600 python bench.py --no-cpu-baseline --steps 20 >> gpurun_out/k0_ab.log 2>&1
done
