mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pipelined or graph or launch_variants or frames_to_host or strip or end_to_end or kernel_timing" > gpurun_out/fold_final.log 2>&1
echo "tests rc=$?" >> gpurun_out/fold_final.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/fold_final.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/fold_bench.log 2>&1
