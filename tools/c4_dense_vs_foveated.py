"""BASELINE config 4: dense render_full (P_b = 1, no reconstruction) vs the foveated path (hifi mask +
sparse march + fp16 W-Net) on 512^3 at 1920x1080 over the 500-frame orbit with the moving gaze of
SURVEY 8(d) (fx = (W-1)/2 + 0.4 W sin(2 pi i/500), fy = (H-1)/2 + 0.4 H sin(4 pi i/500)).
Device times per frame from CUDA events; work from the device sample counters.
usage: python tools/c4_dense_vs_foveated.py [frames=500] [out.json]"""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_09965_b200 import network as N  # noqa: E402
from paper_2209_09965_b200.noise import default_stack  # noqa: E402
from paper_2209_09965_b200.pipeline import FramePipeline  # noqa: E402
from paper_2209_09965_b200.renderer import OrbitPathSpec, orbit_cameras  # noqa: E402
from paper_2209_09965_b200.sample_maps import HIFI_PRESET, FoveaConfig, pixel_scale_for_film  # noqa: E402
from paper_2209_09965_b200.throughput import default_scene  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 500
out = Path(sys.argv[2]) if len(sys.argv) > 2 else None
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


ctx = pipe.ctx
s = ctx.stream
# warm-up: textures, workspaces, and the marcher's record buffer grown to the orbit's largest
# frames (every 5th frame, dense and foveated) so the timed pass measures the steady state
for i in range(0, frames, 5):
    pipe.dense(cams[i])
    pipe.step(cams[i], gaze(i), i)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
dense_ms, dense_samples, fov_ms, march_ms, fov_samples, rays = [], [], [], [], [], []
for i in range(frames):
    ctx.reset_stats()
    ev[0].record(s)
    pipe.dense(cams[i])
    ev[1].record(s)
    ev[1].synchronize()
    st = ctx.stats()
    dense_ms.append(ev[0].elapsed_time(ev[1]))
    dense_samples.append(st.samples_main + st.samples_shadow)
    ctx.reset_stats()
    m_ms, r_ms, n_ms = pipe.step(cams[i], gaze(i), i, timed=True)
    st = ctx.stats()
    fov_ms.append(m_ms + r_ms + n_ms)
    march_ms.append(m_ms + r_ms)
    fov_samples.append(st.samples_main + st.samples_shadow)
    rays.append(st.rays)
res = {
    "config": "C4: 512^3 sphere_shells, 1920x1080, orbit of 500 frames, moving gaze, hifi (P_b=0.07, sigma=0.06)",
    "frames": frames,
    "dense_ms_mean": float(np.mean(dense_ms)), "dense_fps": 1e3 / float(np.mean(dense_ms)),
    "dense_samples_per_frame": float(np.mean(dense_samples)),
    "foveated_ms_mean": float(np.mean(fov_ms)), "foveated_fps": 1e3 / float(np.mean(fov_ms)),
    "foveated_mask_march_ms_mean": float(np.mean(march_ms)),
    "foveated_samples_per_frame": float(np.mean(fov_samples)), "foveated_rays_per_frame": float(np.mean(rays)),
    "speedup_total": float(np.mean(dense_ms) / np.mean(fov_ms)),
    "speedup_render_only": float(np.mean(dense_ms) / np.mean(march_ms)),
    "sample_ratio": float(np.mean(dense_samples) / np.mean(fov_samples)),
    "timing": "serial per frame, CUDA events on the pipeline stream",
}
print(json.dumps(res, indent=1))
if out:
    out.write_text(json.dumps(res, indent=1) + "\n")
