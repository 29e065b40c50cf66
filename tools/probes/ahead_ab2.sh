mkdir -p gpurun_out
for rep in 1 2; do
for k in 0 5 6 7 8 9 10 12; do
  echo "== FV_MARCH_AHEAD=$k" >> gpurun_out/ahead_ab2.log
  FV_MARCH_AHEAD=$k timeout 600 python bench.py --no-cpu-baseline --steps 40 >> gpurun_out/ahead_ab2.log 2>&1
done
done
