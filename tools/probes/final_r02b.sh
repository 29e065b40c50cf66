# round-2 final evidence (after the double-buffered, folded filter chain)
set -x
mkdir -p gpurun_out
FV_PARITY_REPORT=gpurun_out/r02_headline_parity.json timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fin_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin_bench.log 2>&1; echo "rc=$?" >> gpurun_out/fin_bench.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/fin_bench2.log 2>&1
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin_ref.log 2>&1; echo "rc=$?" >> gpurun_out/fin_ref.log
for c in c1 c2; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/fin_cfg_$c.log 2>&1; done
timeout 900 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/fin_cfg_c5.log 2>&1
timeout 600 python tools/probes/timeline.py > gpurun_out/fin_timeline.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/fin_ncu_launches.log 2>&1
