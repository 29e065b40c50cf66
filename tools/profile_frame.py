"""Run a few C3 frames through the device pipeline (for ncu launch lists / captures)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import CONFIGS, PATH_FRAMES  # noqa: E402
from paper_2209_09965_b200 import network as N  # noqa: E402
from paper_2209_09965_b200.noise import default_stack  # noqa: E402
from paper_2209_09965_b200.pipeline import FramePipeline  # noqa: E402
from paper_2209_09965_b200.renderer import OrbitPathSpec, orbit_cameras  # noqa: E402
from paper_2209_09965_b200.sample_maps import FoveaConfig, pixel_scale_for_film  # noqa: E402
from paper_2209_09965_b200.throughput import default_scene  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
h, w, n = cfg["height"], cfg["width"], cfg["vol"]
scene = default_scene("sphere_shells", (n, n, n))
net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
cams = orbit_cameras(OrbitPathSpec(n_frames=PATH_FRAMES), scene.volume, w, h)
fovea = FoveaConfig(focus=((w - 1) / 2.0, (h - 1) / 2.0), sigma=cfg["sigma"], base_density=cfg["pb"],
                    pixel_scale=pixel_scale_for_film((h, w)))
pipe = FramePipeline(scene, net, (h, w), default_stack())
torch.cuda.synchronize()
for i in range(frames):
    pipe.step(cams[i], fovea, i)
torch.cuda.synchronize()
print("frames done", frames)
