mkdir -p gpurun_out
for i in 1 2; do
  timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/soak_$i.log 2>&1
  echo "rc=$?" >> gpurun_out/soak_$i.log
done
for i in 1 2 3; do python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/soak_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/soak_smoke.log; done
