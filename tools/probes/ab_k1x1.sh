# 1x1 (centre-only) K convs without the unused halo rows / columns: parity, then per-class times
timeout 900 python -m pytest tests -m gpu -x -q -k "forward or kernel_stage or conv or end_to_end or graph" > gpurun_out/t_all.log 2>&1; tail -1 gpurun_out/t_all.log
bash tools/probes/ab_libs.sh 3 10 - bench_out/ab/HEAD/libfovnet.so - bench_out/ab/HEAD/libfovnet.so
