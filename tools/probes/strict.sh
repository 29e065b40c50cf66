mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "strict or out_of_range or render" > gpurun_out/strict.log 2>&1
echo "rc=$?" >> gpurun_out/strict.log
