mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "padded" > gpurun_out/padded.log 2>&1
echo "rc=$?" >> gpurun_out/padded.log
