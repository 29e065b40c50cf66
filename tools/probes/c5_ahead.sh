mkdir -p gpurun_out
rm -f gpurun_out/c5_ahead.log
for a in 6 0 6 0 12; do
  echo "== ahead $a" >> gpurun_out/c5_ahead.log
  FV_MARCH_AHEAD=$a timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['timing']['pipelined_ms_per_frame'],3), round(d['timing']['serial_ms_per_frame'],3), d['clocks']['sm_mhz'])" >> gpurun_out/c5_ahead.log
done
