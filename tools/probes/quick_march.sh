mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "render or metrics or pipelined or overflow" > gpurun_out/quick_march.log 2>&1
echo "rc=$?" >> gpurun_out/quick_march.log
