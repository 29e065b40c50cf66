# A/B a library env knob on the C3 bench: bash tools/probes/ab_env.sh "VAR=a" "VAR=b" ...
# (one line per config on stdout and appended to gpurun_out/ab_results.txt)
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$cfg', round(d['value'],1), round(d['timing']['serial_ms_per_frame'],3), round(d['e2e']['value'],1), {n: round(v['ms_per_frame'],3) for n,v in k.items()})" | tee -a gpurun_out/ab_results.txt
done
