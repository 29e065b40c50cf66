"""e2e through fv_frames vs device-only pipelining on the C3 workload."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import CONFIGS, PATH_FRAMES  # noqa: E402
from paper_2209_09965_b200 import network as N  # noqa: E402
from paper_2209_09965_b200.noise import default_stack  # noqa: E402
from paper_2209_09965_b200.pipeline import FramePipeline  # noqa: E402
from paper_2209_09965_b200.renderer import OrbitPathSpec, orbit_cameras  # noqa: E402
from paper_2209_09965_b200.sample_maps import FoveaConfig, pixel_scale_for_film  # noqa: E402
from paper_2209_09965_b200.throughput import default_scene  # noqa: E402

cfg = CONFIGS["c3"]
h, w, n = cfg["height"], cfg["width"], cfg["vol"]
scene = default_scene("sphere_shells", (n, n, n))
net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
cams = orbit_cameras(OrbitPathSpec(n_frames=PATH_FRAMES), scene.volume, w, h)
fovea = FoveaConfig(focus=((w - 1) / 2.0, (h - 1) / 2.0), sigma=cfg["sigma"], base_density=cfg["pb"],
                    pixel_scale=pixel_scale_for_film((h, w)))
pipe = FramePipeline(scene, net, (h, w), default_stack())
pinned = [torch.empty((h, w, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
pageable = [torch.empty((h, w, 3), dtype=torch.float32) for _ in range(2)]
for i in range(3):
    pipe.step(cams[i], fovea, i)
pipe.frames_to_host([(cams[j], fovea, j) for j in range(5)], pinned)
torch.cuda.synchronize()
for nf in (30, 60):
    fr = [(cams[(5 + j) % PATH_FRAMES], fovea, 5 + j) for j in range(nf)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.run_pipelined(fr)
    torch.cuda.synchronize()
    dev = nf / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    pipe.frames_to_host(fr, pinned)
    e2e = nf / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    pipe.frames_to_host(fr, pageable)
    e2e_pg = nf / (time.perf_counter() - t0)
    print(f"{nf} frames: device pipelined {dev:.1f} fps (wall), fv_frames pinned {e2e:.1f}, pageable {e2e_pg:.1f}")
