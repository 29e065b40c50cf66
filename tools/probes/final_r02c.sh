# final round-2 pass: full suite + headline parity report, smoke, bench (C3 default, twice), configs
mkdir -p gpurun_out
FV_PARITY_REPORT=gpurun_out/r02_headline_parity.json timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fz_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fz_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fz_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fz_smoke.log
timeout 900 python bench.py > gpurun_out/fz_bench.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/fz_bench2.log 2>&1
for c in c1 c2; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/fz_cfg_$c.log 2>&1; done
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fz_cfg_c5.log 2>&1
timeout 600 python tools/probes/timeline.py > gpurun_out/fz_timeline.log 2>&1
