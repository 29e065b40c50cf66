# round-2 final evidence: full GPU suite with the headline parity report, the default bench line
# (with its CPU baseline), the reference arm, the bench launch list, a timing of configs
set -x
mkdir -p gpurun_out
FV_PARITY_REPORT=gpurun_out/r02_headline_parity.json timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests_final.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "rc=$?" >> gpurun_out/bench_final.log
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_final.log 2>&1; echo "rc=$?" >> gpurun_out/ref_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
