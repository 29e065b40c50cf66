# row-fused 96-column convs on 2-row tiles (FV_N96_FUSE=1) vs the per-tap issue: shapes, frame conv time, tests
S="176,96,135,240 96,96,135,240"
for v in 0 1 0 1; do echo "== FV_N96_FUSE=$v"; FV_N96_FUSE=$v python tools/probes/conv_bench.py $S; done
for v in 0 1 0 1; do echo "== frame FV_N96_FUSE=$v"; FV_N96_FUSE=$v python tools/probes/kernel_times.py 3 20 | grep -i "conv\|frames"; done
FV_N96_FUSE=1 timeout 900 python -m pytest tests -m gpu -x -q -k "conv or forward or headline_network or pipelined or launch_variants" 2>&1 | tail -2
