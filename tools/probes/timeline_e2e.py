"""CUPTI timeline of the e2e call (fv_frames with pinned host outputs) at C3: where the wall clock
goes beyond the device-timed loop (prologue, D2H copies, tail)."""
import json, sys, time
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
host = [torch.empty((h, w, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
for j in range(5):
    pipe.step(cams[j], fovea, j)
pipe.run_pipelined([(cams[j], fovea, j) for j in range(5)])
pipe.frames_to_host([(cams[j], fovea, j) for j in range(5, 9)], host)
torch.cuda.synchronize()
K = 30
frames = [(cams[9 + j], fovea, 9 + j) for j in range(K)]
for rep in range(2):
    t0 = time.perf_counter()
    pipe.frames_to_host(frames, host)
    print(f"e2e wall {K / (time.perf_counter() - t0):.1f} fps", flush=True)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    pipe.frames_to_host(frames, host)
    wall = time.perf_counter() - t0
print(f"profiled e2e wall {K / wall:.1f} fps ({wall * 1e3:.2f} ms)")
out = Path("gpurun_out"); out.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out / "tl_e2e_raw.json"))
ev = []
for e in json.load(open(out / "tl_e2e_raw.json"))["traceEvents"]:
    if "dur" in e and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime", "cuda_driver", "python_function", "user_annotation", "cpu_op"):
        ev.append({"name": e["name"][:90], "stream": e.get("tid"), "ts": e["ts"], "dur": e["dur"], "cat": e["cat"]})
json.dump(ev, open(out / "tl_e2e.json", "w"))
