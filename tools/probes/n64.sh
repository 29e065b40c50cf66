# 8-row tiles for the streamed-weight 64-column convs (FV_N64_R=8) vs 4-row: isolated shapes, frame conv time
S="208,64,540,960 192,64,1080,1920 256,80,270,480"
for v in 4 8 4 8; do echo "== FV_N64_R=$v"; FV_N64_R=$v python tools/probes/conv_bench.py $S; done
for v in 4 8 4 8; do echo "== frame FV_N64_R=$v"; FV_N64_R=$v python tools/probes/kernel_times.py 3 20 | grep -i "conv\|frames"; done
FV_N64_R=8 timeout 900 python -m pytest tests -m gpu -x -q -k "conv or forward" 2>&1 | tail -2
