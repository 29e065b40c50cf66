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
frames = [(cams[5 + j], fovea, 5 + j) for j in range(16)]
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pipe.run_pipelined(frames)
    torch.cuda.synchronize()
import os
out = Path("gpurun_out"); out.mkdir(exist_ok=True)
tag = os.environ.get("TL_TAG", "")
prof.export_chrome_trace(str(out / f"timeline_raw{tag}.json"))
ev = []
for e in json.load(open(out / f"timeline_raw{tag}.json"))["traceEvents"]:
    if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e:
        ev.append({"name": e["name"][:90], "stream": e.get("tid"), "ts": e["ts"], "dur": e["dur"], "cat": e["cat"]})
json.dump(ev, open(out / f"timeline{tag}.json", "w"))
os.remove(out / f"timeline_raw{tag}.json")
# median frame period on the network stream (E0.conv1 starts)
k = sorted((e for e in ev if e["cat"] == "kernel"), key=lambda e: e["ts"])
net_s = max(set(e["stream"] for e in k), key=lambda s_: sum(1 for e in k if e["stream"] == s_))
# frame boundaries: the per-frame parameter-block copy (HtoD) on the network stream
starts = [e["ts"] for e in sorted(ev, key=lambda e: e["ts"]) if e["cat"] == "gpu_memcpy" and "HtoD" in e["name"]]
per = sorted(b - a for a, b in zip(starts, starts[1:]))
print(f"{tag}: {len(ev)} device events, median frame {per[len(per) // 2]:.1f} us", flush=True)
