# main pass without the inline-shadow fallback in it: register caps (resident blocks per SM)
timeout 900 python -m pytest tests -m gpu -x -q -k "render or sample_counts or c1 or pipelined or overflow or naive or fused or shard" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_libs.sh 3 10 bench_out/ab/HEAD/libfovnet.so bench_out/ab/minb5/libfovnet.so - bench_out/ab/minb7/libfovnet.so bench_out/ab/minb8/libfovnet.so
