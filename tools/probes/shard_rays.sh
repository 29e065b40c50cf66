# strip-sharded frames with the ray-sized record gather: parity tests, then the C5 --shard line
timeout 900 python -m pytest tests -m gpu -x -q -k "shard or strip or records" > gpurun_out/sr_tests.log 2>&1; tail -2 gpurun_out/sr_tests.log
timeout 900 python bench.py --config c5 --shard --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/sr_c5s.log 2>&1; tail -1 gpurun_out/sr_c5s.log | cut -c1-600
