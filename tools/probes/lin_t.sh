mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py -q -m gpu -k "render or march or sample_counts or overflow or pipelined or end_to_end or strict or out_of_range" > gpurun_out/lin_t.log 2>&1
echo "rc=$?" >> gpurun_out/lin_t.log
