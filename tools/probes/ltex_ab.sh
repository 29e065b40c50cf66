# A/B of the filtered texture's texel format (FV_LTEX_BITS 32 = float, 16 = unorm16), then the
# march parity tests with the default (16)
mkdir -p gpurun_out
for b in 32 16 32 16; do
  echo "== bits $b" >> gpurun_out/ltex_ab.log
  FV_LTEX_BITS=$b timeout 600 python bench.py --no-cpu-baseline --steps 20 >> gpurun_out/ltex_ab.log 2>&1
done
timeout 1500 python -m pytest tests/test_headline_parity.py tests/test_gpu_parity.py -q -x -m gpu \
  -k "march or render or sample_counts or end_to_end or overflow" > gpurun_out/ltex_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ltex_tests.log
