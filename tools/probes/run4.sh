# A/B of the marcher's sample source (FV_TEX_FILTER 1 vs 2) + full GPU suite at the default
mkdir -p gpurun_out
for v in "FV_TEX_FILTER=1" "FV_TEX_FILTER=2" "FV_TEX_FILTER=1" "FV_TEX_FILTER=2"; do
  echo "== $v" >> gpurun_out/bench4.log
  env $v timeout 600 python bench.py --no-cpu-baseline >> gpurun_out/bench4.log 2>&1
done
FV_TEX_FILTER=2 FV_PARITY_REPORT=gpurun_out/hp_filter2.json timeout 900 python -m pytest tests/test_headline_parity.py -q -k "C3 and (march or end_to_end)" > gpurun_out/hp_filter2.log 2>&1
FV_PARITY_REPORT=gpurun_out/headline_parity.json timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
