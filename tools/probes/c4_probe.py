"""C4 frames with per-phase times and the marcher's record-buffer feedback (overflow diagnosis).
usage: python tools/probes/c4_probe.py FRAMES"""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2209_09965_b200 import network as N  # noqa: E402
from paper_2209_09965_b200.noise import default_stack  # noqa: E402
from paper_2209_09965_b200.pipeline import FramePipeline  # noqa: E402
from paper_2209_09965_b200.renderer import OrbitPathSpec, orbit_cameras  # noqa: E402
from paper_2209_09965_b200.sample_maps import HIFI_PRESET, FoveaConfig, pixel_scale_for_film  # noqa: E402
from paper_2209_09965_b200.throughput import default_scene  # noqa: E402

frames = int(sys.argv[1])
h, w, n = 1080, 1920, 512
scene = default_scene("sphere_shells", (n, n, n))
net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
cams = orbit_cameras(OrbitPathSpec(n_frames=500), scene.volume, w, h)
pipe = FramePipeline(scene, net, (h, w), default_stack())
scale = pixel_scale_for_film((h, w))


def gaze(i):
    fx = (w - 1) / 2.0 + 0.4 * w * math.sin(2 * math.pi * i / 500)
    fy = (h - 1) / 2.0 + 0.4 * h * math.sin(4 * math.pi * i / 500)
    return FoveaConfig(focus=(fx, fy), sigma=HIFI_PRESET["sigma"], base_density=HIFI_PRESET["base_density"],
                       pixel_scale=scale)


s = pipe.ctx.stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(frames):
    mode = sys.argv[2] if len(sys.argv) > 2 else "both"
    if mode in ("both", "dense"):
        ev[0].record(s)
        pipe.dense(cams[i])
        ev[1].record(s)
        ev[1].synchronize()
        d = ev[0].elapsed_time(ev[1])
    else:
        d = 0.0
    m, r, k = pipe.step(cams[i], gaze(i), i, timed=True)
    print(f"frame {i}: dense {d:.3f} ms  mask {m:.3f} march {r:.3f} net {k:.3f}", flush=True)
