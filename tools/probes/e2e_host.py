"""Host-side cost of frames_to_host: marshalling vs the C call, for 1 and 30 frames."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
from paper_2209_09965_b200 import _lib, network as N
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
dev = [torch.empty((h, w, 3), dtype=torch.float32, device="cuda") for _ in range(2)]
pipe.frames_to_host([(cams[j], fovea, j) for j in range(6)], host)
pipe.run_pipelined([(cams[j], fovea, j) for j in range(6)])
torch.cuda.synchronize()
for K in (1, 30, 30, 30):
    frames = [(cams[10 + j], fovea, 10 + j) for j in range(K)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.frames_to_host(frames, host)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t2 = time.perf_counter()
    e0.record(pipe.ctx.stream)
    pipe.run_pipelined(frames)
    e1.record(pipe.ctx.stream)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"K={K}: host-out call {1e3*(t1-t0):.3f} ms ({K/(t1-t0):.1f} fps); device-out: enqueue {1e3*(t3-t2):.3f} ms, "
          f"wall {1e3*(t4-t2):.3f} ms, events {e0.elapsed_time(e1):.3f} ms", flush=True)
