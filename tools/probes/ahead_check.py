"""fv_frames frames (whatever FV_MARCH_AHEAD / FV_FRAME_GRAPH say) == the serial step-by-step frames."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2209_09965_b200 import network as N  # noqa: E402
from paper_2209_09965_b200.noise import default_stack  # noqa: E402
from paper_2209_09965_b200.pipeline import FramePipeline  # noqa: E402
from paper_2209_09965_b200.renderer import OrbitPathSpec, orbit_cameras  # noqa: E402
from paper_2209_09965_b200.throughput import ExperimentSpec, default_scene  # noqa: E402

spec = ExperimentSpec(mode="hifi", width=320, height=184)
scene = default_scene("sphere_shells", (96, 96, 96))
net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
cams = orbit_cameras(OrbitPathSpec(n_frames=500), scene.volume, 320, 184)
pipe = FramePipeline(scene, net, (184, 320), default_stack())
ref = []
for i in range(8):
    pipe.step(cams[i], spec.fovea(), i)
    ref.append(pipe.rgb.clone())
frames = [(cams[i], spec.fovea(), i) for i in range(8)]
pipe.reset()
outs = [torch.empty_like(pipe.rgb) for _ in range(8)]
pipe.run_pipelined(frames, outs)
torch.cuda.synchronize()
ok = all(torch.equal(outs[i], ref[i]) for i in range(8))
pipe.reset()
for i in range(8):
    pipe.run_pipelined(frames[i:i + 1])
    torch.cuda.synchronize()
    ok &= torch.equal(pipe.rgb, ref[i])
print("IDENTICAL" if ok else "DIFFERENT")
sys.exit(0 if ok else 1)
