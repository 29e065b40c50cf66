# ray setup pass: one list append per block (in-tree) vs per warp (HEAD build)
timeout 900 python -m pytest tests -m gpu -x -q -k "render or sample_counts or c1 or pipelined" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_libs.sh 3 10 - bench_out/ab/HEAD/libfovnet.so - bench_out/ab/HEAD/libfovnet.so
