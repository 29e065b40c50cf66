timeout 900 python -m pytest tests -m gpu -x -q -k "overflow" > gpurun_out/t_ovf.log 2>&1; tail -15 gpurun_out/t_ovf.log
for cfg in "FV_WAVE_REC_PER_RAY=16" "FV_WAVE_REC_PER_RAY=48"; do
  env $cfg timeout 600 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/p.log 2>&1
  tail -1 gpurun_out/p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('c5 $cfg', round(d['value'],1), 'serial', round(d['timing']['serial_ms_per_frame'],3), {n: round(v['ms_per_frame'],3) for n,v in k.items()})"
done
