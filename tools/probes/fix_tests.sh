mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "padded_films or kernel_timing" > gpurun_out/fix_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fix_tests.log
FV_PARITY_REPORT=gpurun_out/headline_parity.json timeout 1200 python -m pytest tests/test_headline_parity.py -q -m gpu >> gpurun_out/fix_tests.log 2>&1
echo "headline rc=$?" >> gpurun_out/fix_tests.log
