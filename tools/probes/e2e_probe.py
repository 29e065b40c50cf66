"""Where does e2e lose to the device-timed frame loop? Repeated 90-frame runs at C3:
run_pipelined (device outputs) vs frames_to_host (pinned host outputs), wall clock and events."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
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
import subprocess, threading
fovea = FoveaConfig(focus=((w - 1) / 2.0, (h - 1) / 2.0), sigma=0.06, base_density=0.07,
                    pixel_scale=pixel_scale_for_film((h, w)))
pipe = FramePipeline(scene, net, (h, w), default_stack(), RenderSettings())
stream = pipe.ctx.stream
host = [torch.empty((h, w, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
dev = [torch.empty((h, w, 3), dtype=torch.float32, device="cuda") for _ in range(2)]
K = 90
for j in range(5):
    pipe.step(cams[j], fovea, j)
torch.cuda.synchronize()
def smi():
    q = "clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,temperature.gpu"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                          capture_output=True, text=True).stdout.strip()
samples = []
stop = False
def poll():
    while not stop:
        samples.append(smi())
threading.Thread(target=poll, daemon=True).start()
for rep in range(4):
    for mode in ("dev", "host", "host1"):
        frames = [(cams[(j + 25) % 500], fovea, j) for j in range(K)]
        pipe.ctx.reset_stats()
        samples.clear()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record(stream)
        if mode == "dev":
            pipe.run_pipelined(frames)
        elif mode == "host":
            pipe.frames_to_host(frames, host)
        else:
            pipe.frames_to_host(frames, host[:1])
        e1.record(stream); torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st = pipe.ctx.stats()
        print(f"rep {rep} {mode:5s}: wall {K / wall:7.1f} fps  events {K / (e0.elapsed_time(e1) / 1e3):7.1f} fps"
              f"  rays/frame {st.rays / K:.0f}  smi {samples[-3:]}", flush=True)
stop = True
for K in (20, 40, 90, 200):
    frames = [(cams[(j + 5) % 500], fovea, j) for j in range(K)]
    torch.cuda.synchronize(); time.sleep(1.0)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream); pipe.run_pipelined(frames); e1.record(stream); torch.cuda.synchronize()
    print(f"after 1 s idle, {K} frames: {K / (e0.elapsed_time(e1) / 1e3):7.1f} fps", flush=True)
K = 90
# copy alone: 90 D2H copies of one frame
torch.cuda.synchronize()
t0 = time.perf_counter()
for j in range(K):
    host[j & 1].copy_(dev[0], non_blocking=True)
torch.cuda.synchronize()
print(f"D2H alone: {(time.perf_counter() - t0) / K * 1e3:.3f} ms per frame ({h*w*12/1e6:.1f} MB)")
