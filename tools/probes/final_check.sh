mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fc_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fc_smoke.log
timeout 900 python bench.py > gpurun_out/fc_bench.log 2>&1
