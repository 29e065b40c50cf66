# kapply_pool register cap: in-tree (no cap) vs bench_out/ab/kpool8 (64 registers)
bash tools/probes/ab_libs.sh 3 10 - bench_out/ab/kpool8/libfovnet.so - bench_out/ab/kpool8/libfovnet.so
