# every BASELINE config on one B200 (C4 via its own tool); one JSON summary line each
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cfg_$c.log 2>&1
  tail -1 gpurun_out/cfg_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'serial', round(d['timing']['serial_ms_per_frame'],3), 'phases', {k: round(v,3) for k,v in d['phase_ms'].items()}, 'march Gs/s', round(d['stages']['march']['gsamples_per_s'],1), 'frac', round(d['stages']['march']['frac'],3), 'e2e', round(d['e2e']['value'],1))" | tee -a gpurun_out/cfg_results.txt
done
timeout 900 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c5.log 2>&1
tail -1 gpurun_out/cfg_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value'],1), 'serial', round(d['timing']['serial_ms_per_frame'],3), 'phases', {k: round(v,3) for k,v in d['phase_ms'].items()}, 'march Gs/s', round(d['stages']['march']['gsamples_per_s'],1), 'frac', round(d['stages']['march']['frac'],3), 'e2e', round(d['e2e']['value'],1))" | tee -a gpurun_out/cfg_results.txt
timeout 900 python bench.py --config c5 --shard --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c5s.log 2>&1; tail -1 gpurun_out/cfg_c5s.log | cut -c1-400 | tee -a gpurun_out/cfg_results.txt
timeout 1200 python tools/c4_dense_vs_foveated.py > gpurun_out/c4.log 2>&1; tail -5 gpurun_out/c4.log | tee -a gpurun_out/cfg_results.txt
