mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/tests_only.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests_only.log
FV_PARITY_REPORT=gpurun_out/headline_parity.json timeout 900 python -m pytest tests/test_headline_parity.py -q -m gpu > /dev/null 2>&1
