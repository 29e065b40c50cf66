mkdir -p gpurun_out
FV_SHADOW_FILTER=1 FV_PARITY_REPORT=gpurun_out/hp_filter.json timeout 900 python -m pytest tests/test_headline_parity.py -q -k "C3 and (march or end_to_end)" > gpurun_out/hp_filter.log 2>&1
for v in "" "FV_SHADOW_FILTER=1" "FV_SHADOW_FILTER=1 FV_SHADOW_LIN_U=8"; do
  echo "== $v" >> gpurun_out/bench3.log
  env $v timeout 600 python bench.py --no-cpu-baseline >> gpurun_out/bench3.log 2>&1
done
