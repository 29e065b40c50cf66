# default bench twice + per-launch frame list
timeout 600 python -m pytest tests -m gpu -x -q -k "overflow or launch_variants" 2>&1 | tail -1
for i in 1 2; do python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), round(d['roofline']['achieved'],1), d['roofline']['peak'])"; done
FV_KTIME_LOG=1 python tools/probes/kernel_times.py 3 16 2> gpurun_out/qb_spans.log | grep -v "^ *$"; python tools/probes/launch_times.py gpurun_out/qb_spans.log 16
