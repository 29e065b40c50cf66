"""Per-launch device times (CUDA events around each launch) averaged over C3 frames, in launch
order. usage: FV_KTIME_LOG=1 python tools/probes/kernel_times.py 10 8 2> spans.log;
python tools/probes/launch_times.py spans.log 8"""
import sys
from collections import defaultdict

CLS = {0: "mask", 1: "march_main", 2: "march_shadow", 3: "march_composite", 4: "conv", 5: "netops", 6: "other"}
rows = [ln.split()[1:] for ln in open(sys.argv[1]) if ln.startswith("[kspan]")]
frames = int(sys.argv[2])
per = len(rows) // frames
acc = defaultdict(float)
for i, (c, w, t) in enumerate(rows[: per * frames]):
    acc[i % per] += float(t) * 1e3 / frames
tot = 0.0
for i in range(per):
    c, w, _ = rows[i]
    tf = float(w) / (acc[i] * 1e-6) / 1e12 if float(w) > 0 else 0.0
    tot += acc[i]
    print(f"{i:3d} {CLS.get(int(c), c):16s} {acc[i]:8.1f} us" + (f"  {tf:7.1f} TFLOP/s" if tf else ""))
print(f"sum {tot:.1f} us per frame ({per} launches)")
