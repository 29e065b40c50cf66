mkdir -p gpurun_out
for k in 0 2 4 6 8; do
  echo "== FV_MARCH_AHEAD=$k" >> gpurun_out/ahead_ab.log
  FV_MARCH_AHEAD=$k timeout 300 python tools/probes/ahead_check.py >> gpurun_out/ahead_ab.log 2>&1
  FV_MARCH_AHEAD=$k timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/ahead_ab.log 2>&1
done
