mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "launch_variants" > gpurun_out/variants.log 2>&1
echo "rc=$?" >> gpurun_out/variants.log
