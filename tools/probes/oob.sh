mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "out_of_range or render or c1 or pipelined or padded or end_to_end" > gpurun_out/oob.log 2>&1
echo "rc=$?" >> gpurun_out/oob.log
timeout 300 python tools/probes/oob_probe.py >> gpurun_out/oob.log 2>&1
