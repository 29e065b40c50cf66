"""Per-kernel-class device times (CUDA events around each launch) for frames [first, first+count)
of the C3 orbit, serial order. usage: python tools/probes/kernel_times.py FIRST COUNT [c3|c2]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import CONFIGS, PATH_FRAMES  # noqa: E402
from paper_2209_09965_b200 import _lib  # noqa: E402
from paper_2209_09965_b200 import network as N  # noqa: E402
from paper_2209_09965_b200.noise import default_stack  # noqa: E402
from paper_2209_09965_b200.pipeline import FramePipeline  # noqa: E402
from paper_2209_09965_b200.renderer import OrbitPathSpec, orbit_cameras  # noqa: E402
from paper_2209_09965_b200.sample_maps import FoveaConfig, pixel_scale_for_film  # noqa: E402
from paper_2209_09965_b200.throughput import default_scene  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
cfg = CONFIGS[sys.argv[3] if len(sys.argv) > 3 else "c3"]
h, w, n = cfg["height"], cfg["width"], cfg["vol"]
scene = default_scene("sphere_shells", (n, n, n))
net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
cams = orbit_cameras(OrbitPathSpec(n_frames=PATH_FRAMES), scene.volume, w, h)
fovea = FoveaConfig(focus=((w - 1) / 2.0, (h - 1) / 2.0), sigma=cfg["sigma"], base_density=cfg["pb"],
                    pixel_scale=pixel_scale_for_film((h, w)))
pipe = FramePipeline(scene, net, (h, w), default_stack())
for j in range(3):
    pipe.step(cams[j], fovea, j)
torch.cuda.synchronize()
ctx = pipe.ctx
ctx.reset_stats()
ctx.set_kernel_timing(True)
for j in range(first, first + count):
    pipe.step(cams[j % PATH_FRAMES], fovea, j)
torch.cuda.synchronize()
st = ctx.stats()
res = {k: ctx.kernel_time(c) for k, c in _lib.KERNEL_CLASSES.items()}
print(f"frames {first}..{first + count - 1}: rays/frame {st.rays / count:.0f} hits/frame {st.hit_rays / count:.0f} main samples/frame "
      f"{st.samples_main / count / 1e6:.2f} M shadow samples/frame {st.samples_shadow / count / 1e6:.2f} M")
for k, (ms, work, nl) in res.items():
    if nl:
        print(f"  {k:16s} {ms / count * 1e3:9.1f} us/frame  ({nl / count:.0f} launches/frame)")
