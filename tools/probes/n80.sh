# 4-row tiles for the 80-column convs (FV_N80_R=4) vs the 2-row default: isolated shapes, frame conv time, tests
S="256,80,270,480 64,80,270,480 80,80,270,480"
for v in 2 4 2 4; do echo "== FV_N80_R=$v"; FV_N80_R=$v python tools/probes/conv_bench.py $S; done
for v in 2 4 2 4; do echo "== frame FV_N80_R=$v"; FV_N80_R=$v python tools/probes/kernel_times.py 3 20 | grep -i "conv\|frames"; done
FV_N80_R=4 timeout 900 python -m pytest tests -m gpu -x -q -k "conv or forward or headline_network or pipelined" 2>&1 | tail -2
