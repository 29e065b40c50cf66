# graph replay priority: C5 and C3 pipelined with and without graphs
for cfg in "FV_GRAPH=1" "FV_GRAPH=0"; do
  env $cfg timeout 600 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/p.log 2>&1
  tail -1 gpurun_out/p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $cfg', round(d['value'],1), 'serial', round(d['timing']['serial_ms_per_frame'],3), 'e2e', round(d['e2e']['value'],1))" | tee -a gpurun_out/ab_results.txt
done
bash tools/probes/ab_env.sh "FV_GRAPH=1" "FV_GRAPH=0" "FV_GRAPH=1" "FV_GRAPH=0"
