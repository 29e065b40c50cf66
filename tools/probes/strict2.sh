mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "strict" > gpurun_out/strict2.log 2>&1
echo "rc=$?" >> gpurun_out/strict2.log
FV_TEX_FILTER=0 timeout 600 python bench.py --no-cpu-baseline --no-sustained --steps 20 2>/dev/null | tail -1 | cut -c1-160 >> gpurun_out/strict2.log
timeout 600 python bench.py --no-cpu-baseline --no-sustained --steps 20 2>/dev/null | tail -1 | cut -c1-160 >> gpurun_out/strict2.log
