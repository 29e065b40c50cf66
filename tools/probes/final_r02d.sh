# final check of the round's code: full GPU suite + headline parity report, smoke, bench twice
mkdir -p gpurun_out
FV_PARITY_REPORT=gpurun_out/r02_headline_parity.json timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fd_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fd_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fd_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fd_smoke.log
timeout 900 python bench.py > gpurun_out/fd_bench.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/fd_bench2.log 2>&1
