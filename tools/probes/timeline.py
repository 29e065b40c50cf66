"""Kernel timeline of the C3 frame loop (CUPTI via torch.profiler): which kernels overlap, and
how much of each frame the network / march branches are exposed. Writes gpurun_out/timeline.json
(kernel name, stream, start/end us) for offline analysis."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2209_09965_b200 import network as N
from paper_2209_09965_b200.noise import default_stack
from paper_2209_09965_b200.pipeline import FramePipeline
from paper_2209_09965_b200.renderer import OrbitPathSpec, RenderSettings, orbit_cameras
from paper_2209_09965_b200.sample_maps import FoveaConfig, pixel_scale_for_film
from paper_2209_09965_b200.throughput import default_scene

h, w, n = 1080, 1920, 512
scene = default_scene("sphere_shells", (n, n, n))
net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
cams = orbit_cameras(OrbitPathSpec(n_frames=500), scene.volume, w, h)
fovea = FoveaConfig(focus=((w - 1) / 2.0, (h - 1) / 2.0), sigma=0.06, base_density=0.07,
                    pixel_scale=pixel_scale_for_film((h, w)))
pipe = FramePipeline(scene, net, (h, w), default_stack(), RenderSettings())
for j in range(5):
    pipe.step(cams[j], fovea, j)
pipe.run_pipelined([(cams[j], fovea, j) for j in range(5)])
torch.cuda.synchronize()
frames = [(cams[5 + j], fovea, 5 + j) for j in range(12)]
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pipe.run_pipelined(frames)
    torch.cuda.synchronize()
out = Path("gpurun_out"); out.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out / "timeline_raw.json"))
ev = []
for e in json.load(open(out / "timeline_raw.json"))["traceEvents"]:
    if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e:
        ev.append({"name": e["name"][:90], "stream": e.get("tid"), "ts": e["ts"], "dur": e["dur"], "cat": e["cat"]})
json.dump(ev, open(out / "timeline.json", "w"))
print(len(ev), "device events")
