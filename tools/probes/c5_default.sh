mkdir -p gpurun_out
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained 2>/dev/null | tail -1 | cut -c1-200 > gpurun_out/c5_default.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sustained 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/c5_default.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pipelined or launch_variants" >> gpurun_out/c5_default.log 2>&1
