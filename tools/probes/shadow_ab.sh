# A/B of the filtered shadow pass's (samples in flight, blocks/SM); kernel times from bench's timing pass
mkdir -p gpurun_out
for c in 4,8 8,8 4,12 8,12 4,16 6,10; do
  echo "== $c" >> gpurun_out/shadow_ab.log
  FV_SHADOW_LIN=$c timeout 600 python bench.py --no-cpu-baseline --steps 20 >> gpurun_out/shadow_ab.log 2>&1
done
