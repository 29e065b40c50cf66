#!/usr/bin/env python
"""Headline benchmark: foveated render + reconstruct frames/s at 1080p on B200.

Workload (BASELINE.json configs[2], the north-star target; `--config c2` selects configs[1]):
  512^3 sphere_shells volume, 1920x1080 film, 'hifi' preset (P_b=0.07, sigma=0.06),
  FULL_BLOCKS W-Net (seed 0, fp16 weights), orbit camera path of 500 frames, noise frame i,
  recurrent state carried across frames -- one `step` = one frame of
  bench.cmd_bench_throughput's loop body (mask -> compact -> march -> reconstruct).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c2]

Multi-GPU (torchrun, one process per GPU): every rank renders its own frame stream (an
independent viewer session) -- the per-frame path has no exchange step, so there is no
data-path collective; `value` is all ranks' frames / the max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c3": dict(vol=512, width=1920, height=1080, mode="hifi", pb=0.07, sigma=0.06,
               name="512^3 sphere_shells, 1920x1080, hifi (P_b=0.07, sigma=0.06), FULL_BLOCKS fp16 net"),
    "c2": dict(vol=256, width=1920, height=1080, mode="fast", pb=0.03, sigma=0.02,
               name="256^3 sphere_shells, 1920x1080, fast (P_b=0.03, sigma=0.02), FULL_BLOCKS fp16 net"),
    "c1": dict(vol=64, width=256, height=256, mode="fast", pb=0.03, sigma=0.02,
               name="64^3 sphere_shells, 256x256, fast (P_b=0.03, sigma=0.02), FULL_BLOCKS fp16 net"),
    "c5": dict(vol=1024, width=3840, height=2160, mode="fast", pb=0.03, sigma=0.02,
               name="1024^3 sphere_shells, 3840x2160, fast (P_b=0.03, sigma=0.02), FULL_BLOCKS fp16 net"),
}
PATH_FRAMES = 500
MAC_PER_PX = 275071.5  # FULL_BLOCKS multiply-accumulates per output pixel
BYTES_PER_SAMPLE = 32  # algorithmic bytes of one trilinear sample (2x2x2 fp32 footprint)
METRIC = "frames/sec at 1080p (render+reconstruct)"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def device_memory_gb():
    """Device memory in use on this GPU (all allocations of the process: volume, textures, marcher
    workspace, network state), GB."""
    import torch

    free, total = torch.cuda.mem_get_info()
    return round((total - free) / 1e9, 2)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# FV_DIST_BACKEND=gloo: a functional check of the torchrun path on a box with fewer GPUs than ranks
# (ranks share devices round-robin, timing all-reduces go through host tensors). Never for numbers.
DIST_BACKEND = os.environ.get("FV_DIST_BACKEND", "nccl")


def init_rank_device(local: int, world: int):
    """Bind this rank's GPU and join the process group; returns the device for timing all-reduces."""
    import torch

    dev = local % torch.cuda.device_count() if DIST_BACKEND == "gloo" else local
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist

        if DIST_BACKEND == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    return "cuda" if DIST_BACKEND == "nccl" else None


RANK_STRIDE = 977  # each rank's session starts at its own point of the camera path / noise loop


def rank_frames(rank: int, start: int, count: int) -> list[int]:
    """Frame indices rank `rank` renders: its own stream (path frame = index % PATH_FRAMES)."""
    return [rank * RANK_STRIDE + start + i for i in range(count)]


def max_over_ranks(value: float, world: int, device=None) -> float:
    """All-reduce MAX of a per-rank time (device tensor under NCCL, CPU tensor under gloo)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank: int, world: int, max_seconds: float) -> float:
    return world * units_per_rank / max_seconds


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 20 ms around the timed region."""

    def __init__(self, device: int, out: Path):
        self.out = out
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(out, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait(timeout=10)
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------ CPU legs
class CpuFrames:
    """The reference's per-frame loop body (bench.py:194-209) on the host, restated by the oracle:
    NumPy fp64 mask + compaction, the C fp64 marcher over ALL active rays on every host thread,
    and the fp32 NumPy/BLAS W-Net (FULL_BLOCKS, seed 0, fp16-rounded weights) at the full film with
    the recurrent state carried -- whole frames, nothing extrapolated."""

    def __init__(self, cfg):
        from oracle import fovray_oracle as O

        self.O, self.cfg = O, cfg
        self.blas_threads = None  # the BLAS pool's size during the timed frames
        h, w, n = cfg["height"], cfg["width"], cfg["vol"]
        self.stack = O.load_rnkstack(ROOT / "paper_2209_09965_b200" / "data" / "stbn_64x64x8_s1.noise")
        self.tau = O.tau_map(h, w, ((w - 1) / 2, (h - 1) / 2), cfg["sigma"], cfg["pb"], O.pixel_scale_for_film(h, w))
        self.vol = _oracle_volume(n)
        self.params = O.init_params(O.FULL_BLOCKS, 0, fp16_weights=True)
        self.state = None
        self.rays = 0

    def frame(self, i):
        """One frame; returns (seconds, (mask, march, net) seconds)."""
        if self.blas_threads is None:
            self.blas_threads = blas_threads()
        O, cfg = self.O, self.cfg
        h, w, n = cfg["height"], cfg["width"], cfg["vol"]
        t0 = time.perf_counter()
        bits = O.sample_mask(self.stack, h, w, i, self.tau)
        idx = O.compact(bits)
        t1 = time.perf_counter()
        pos, look = O.orbit_camera(i % PATH_FRAMES, PATH_FRAMES, (n, n, n))
        rgba, _ = O.render(self.vol, (1, 1, 1), O.DEFAULT_LUT, ("dir", (-1.0, -1.0, -0.5), (1, 1, 1)),
                           dict(position=pos, look_at=look, fov_y=45.0, width=w, height=h), pix=idx)
        t2 = time.perf_counter()
        img = np.zeros((h * w, 4), np.float32)
        img[idx] = rgba
        m = bits.astype(np.float32)
        x = np.concatenate([np.moveaxis(img.reshape(h, w, 4), -1, 0) * m[None], m[None]], 0)
        o, _, self.state = O.net_forward(self.params, O.FULL_BLOCKS, x, self.state)
        np.clip(o, 0.0, 1.0)
        t3 = time.perf_counter()
        self.rays += int(idx.size)
        return t3 - t0, (t1 - t0, t2 - t1, t3 - t2)

    def describe(self, frames, phases):
        ph = np.mean(np.asarray(phases), axis=0) if phases else (0, 0, 0)
        if self.blas_threads is None:
            self.blas_threads = blas_threads()
        return (f"{frames} whole frames of the reference loop body restated by the oracle (NumPy fp64 mask, C fp64 "
                f"marcher on all {len(os.sched_getaffinity(0))} host threads over all active rays, NumPy/BLAS "
                f"fp32 FULL_BLOCKS net at the full film, state carried): mean mask {ph[0]*1e3:.0f} ms, march "
                f"{ph[1]:.2f} s, net {ph[2]:.2f} s per frame; CPU {cpu_model()}; BLAS threads "
                f"{self.blas_threads}; OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS', 'unset')}, "
                f"OMP_NUM_THREADS={os.environ.get('OMP_NUM_THREADS', 'unset')}")


def blas_threads():
    """Threads of the BLAS pool NumPy uses right now (threadpoolctl)."""
    from threadpoolctl import threadpool_info

    n = [p.get("num_threads") for p in threadpool_info() if p.get("user_api") == "blas"]
    return n[0] if n else None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_frame_sample(cfg, frames=2):
    """cpu_baseline of the GPU arm: a bounded sample -- `frames` whole frames (~10-30 s)."""
    cf = CpuFrames(cfg)
    secs, phases = [], []
    for i in range(frames):
        s_, ph = cf.frame(i)
        secs.append(s_)
        phases.append(ph)
    return float(np.mean(secs)), cf.describe(frames, phases), len(os.sched_getaffinity(0))


_VOL_CACHE = {}


def _oracle_volume(n):
    """The procedural volume for the CPU legs (generated once; the oracle's own generator)."""
    if n not in _VOL_CACHE:
        from oracle import fovray_oracle as O

        _VOL_CACHE[n], _ = O.procedural_volume("sphere_shells", (n, n, n)) if n <= 256 else \
            _procedural_by_slabs(n)
    return _VOL_CACHE[n]


def _procedural_by_slabs(n):
    """sphere_shells at n^3 without the fp64 full-volume temporaries (same values as the oracle)."""
    ax = (np.arange(n) + 0.5) / n * 2.0 - 1.0
    out = np.empty((n, n, n), np.float32)
    lo, hi = np.inf, -np.inf
    raws = []
    for z in range(n):
        r = np.sqrt(ax[None, :] ** 2 + ax[:, None] ** 2 + ax[z] ** 2)
        raw = 0.5 * (1.0 + np.cos(2.0 * np.pi * 3.0 * r))
        lo, hi = min(lo, raw.min()), max(hi, raw.max())
        raws.append(raw)
    for z in range(n):
        out[z] = ((raws[z] - lo) / (hi - lo)).astype(np.float32)
    return out, (lo, hi)


def run_reference(args, cfg):
    """The reference arm: the reference's CPU path (restated by the oracle port) timed on whole
    frames on the host cores -- W warm-up frames, then K timed frames of the carried sequence."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    k, wu = args.steps, args.warmup
    cf = CpuFrames(cfg)
    per, phases = [], []
    # torchrun sets OMP_NUM_THREADS=1 for every rank; rank 0 alone runs this arm, so the BLAS pool
    # is raised to every host thread it may use (the C marcher sizes itself from the affinity mask)
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=len(os.sched_getaffinity(0))):
        for s_ in range(wu + k):
            sec, ph = cf.frame(s_)
            if s_ >= wu:
                per.append(sec)
                phases.append(ph)
    fps = 1.0 / float(np.mean(per))
    threads = len(os.sched_getaffinity(0))
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus, "steps": k,
            "warmup": wu, "ms_per_step": float(np.mean(per)) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp64 (march) / fp32 (net)",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["name"], "film": [cfg["width"], cfg["height"]],
                       "volume": [cfg["vol"]] * 3, "path_frames": PATH_FRAMES, "parallelism": "host threads"},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": cf.describe(k, phases)},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU leg
def run_ours(args, cfg):
    import torch

    rank, world, local = dist_env()
    tdev = init_rank_device(local, world)
    from paper_2209_09965_b200 import _lib
    from paper_2209_09965_b200 import network as N
    from paper_2209_09965_b200.noise import default_stack
    from paper_2209_09965_b200.pipeline import FramePipeline
    from paper_2209_09965_b200.renderer import OrbitPathSpec, RenderSettings, orbit_cameras
    from paper_2209_09965_b200.sample_maps import FoveaConfig, pixel_scale_for_film
    from paper_2209_09965_b200.throughput import default_scene

    h, w, n = cfg["height"], cfg["width"], cfg["vol"]
    scene = default_scene("sphere_shells", (n, n, n))
    net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
    cams = orbit_cameras(OrbitPathSpec(n_frames=PATH_FRAMES), scene.volume, w, h)
    fovea = FoveaConfig(focus=((w - 1) / 2.0, (h - 1) / 2.0), sigma=cfg["sigma"], base_density=cfg["pb"],
                        pixel_scale=pixel_scale_for_film((h, w)))
    pipe = FramePipeline(scene, net, (h, w), default_stack(), RenderSettings())
    ctx = pipe.ctx
    stream = ctx.stream
    k, wu = args.steps, args.warmup
    # clocks are sampled (every 20 ms) from the start of warm-up to the end of the timed region
    clocks = ClockSampler(local, ROOT / "gpurun_out" / f"clocks_r{rank}.csv") if rank == 0 else None
    for j in rank_frames(rank, 0, wu):
        pipe.step(cams[j % PATH_FRAMES], fovea, j)
    pipe.run_pipelined([(cams[j % PATH_FRAMES], fovea, j) for j in rank_frames(rank, 0, wu)])
    torch.cuda.synchronize()
    timed_frames = rank_frames(rank, wu, k)
    # --- device-resident timed region 1: the headline, the frame loop (run_pipelined) ---
    # (mask + march of frame t+1 on one stream while frame t reconstructs on the other)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    lp0 = sum(c.launches() for c in pipe.pipelined_contexts())
    p_start = torch.cuda.Event(enable_timing=True)
    p_end = torch.cuda.Event(enable_timing=True)
    p_start.record(stream)
    pipe.run_pipelined([(cams[j % PATH_FRAMES], fovea, j) for j in timed_frames])
    p_end.record(stream)
    torch.cuda.synchronize()
    launches = sum(c.launches() for c in pipe.pipelined_contexts()) - lp0
    pipe_ms = max_over_ranks(p_start.elapsed_time(p_end), world, device=tdev)
    # --- timed region E (right after region 1, the same K frames): end to end through the C ABI
    # with host buffers (fv_frames): every frame's camera + fovea go in by value and its (H,W,3)
    # f32 image comes back into pinned host memory ---
    host = [torch.empty((h, w, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
    ke = k
    # (4 warm-up frames: both buffer parities run once eagerly and are then captured as graphs)
    pipe.frames_to_host([(cams[j % PATH_FRAMES], fovea, j) for j in rank_frames(rank, wu + k, 4)], host)
    e2e_frames = [(cams[j % PATH_FRAMES], fovea, j) for j in rank_frames(rank, wu + k + 4, ke)]
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    pipe.frames_to_host(e2e_frames, host)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world, device=tdev)
    e2e_fps = whole_job_rate(ke, world, e2e_s)
    # --- timed region 2: the same frames serialised on one stream, with per-phase events ---
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(k)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ctx.reset_stats()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i, j in enumerate(timed_frames):
        e = ev[i]
        e[0].record(stream)
        pipe.mask(fovea, j)
        e[1].record(stream)
        pipe.march(cams[j % PATH_FRAMES])
        e[2].record(stream)
        pipe.reconstruct()
        e[3].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    serial_ms = max_over_ranks(t_start.elapsed_time(t_end), world, device=tdev)
    st = ctx.stats()  # work counters of region 2 only
    # --- timed region 3: the same frames again with CUDA events around every library launch
    # (per-kernel-class launch durations for the roofline; kept out of regions 1 and 2) ---
    ctx.set_kernel_timing(True)
    for j in timed_frames:
        pipe.mask(fovea, j)
        pipe.march(cams[j % PATH_FRAMES])
        pipe.reconstruct()
    torch.cuda.synchronize()
    kern = {name: ctx.kernel_time(cls) for name, cls in _lib.KERNEL_CLASSES.items()}
    ctx.set_kernel_timing(False)
    elapsed_ms = pipe_ms
    clk = clocks.stop() if clocks else None
    mask_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    march_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    net_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    samples_per_frame = (st.samples_main + st.samples_shadow) / k
    rays_per_frame = st.rays / k
    fps = whole_job_rate(k, world, elapsed_ms / 1e3)
    # the same frames one blocking fv_frame call at a time (no overlap of copy and compute)
    t0 = time.perf_counter()
    for c, f, j in e2e_frames[: max(3, ke // 2)]:
        pipe.frame_to_host(c, f, j, host[0])
    e2e_serial_fps = whole_job_rate(max(3, ke // 2), world, max_over_ranks(time.perf_counter() - t0, world,
                                                                           device=tdev))
    # --- sustained (reported, not the headline): a ~1 s device-resident run of the same loop with
    # its own clock record -- the B200 reaches its board power limit within ~0.1 s of this load,
    # after which the SM clock settles below max (sw_power_cap) ---
    sustained = None
    if not args.no_sustained:
        n_sus = max(k, int(1.0 / max(elapsed_ms / k / 1e3, 1e-4)))
        sus_clk = ClockSampler(local, ROOT / "gpurun_out" / f"clocks_sustained_r{rank}.csv") if rank == 0 else None
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        pipe.run_pipelined([(cams[j % PATH_FRAMES], fovea, j) for j in rank_frames(rank, 0, n_sus)])
        s1.record(stream)
        torch.cuda.synchronize()
        sus_ms = max_over_ranks(s0.elapsed_time(s1), world, device=tdev)
        sustained = {"frames": n_sus, "value": whole_job_rate(n_sus, world, sus_ms / 1e3), "unit": "frames/s",
                     "ms_per_frame": sus_ms / n_sus, "clocks": sus_clk.stop() if sus_clk else None}
    h2d = C.sizeof(_lib.FvCamera) + C.sizeof(_lib.FvFovea) + C.sizeof(C.c_int)
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    hbm, tf_burst, tf_sus, src = load_peaks()
    # the tensor denominator follows the measured clock: a region that ran at the maximum SM clock
    # (median >= 95% of max) is judged against the BURST dense peak, otherwise the sustained one
    at_max = bool(clk and clk.get("sm_mhz") and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"])
    tf_sus_raw = tf_sus
    if at_max:
        tf_sus = tf_burst
    peak_kind = "burst dense fp16/bf16, SM clock at max" if at_max else "sustained dense fp16/bf16"
    march_gbs = samples_per_frame * BYTES_PER_SAMPLE / (march_ms / 1e3) / 1e9
    net_tflops = 2 * MAC_PER_PX * h * w / (net_ms / 1e3) / 1e12
    stages = {
        "march": {"bound": "hbm", "achieved": march_gbs, "peak": hbm, "unit": "GB/s",
                  "frac": march_gbs / hbm, "ms": march_ms, "gsamples_per_s": samples_per_frame / (march_ms / 1e3) / 1e9},
        "reconstruct": {"bound": "tensor", "achieved": net_tflops, "peak": tf_sus, "unit": "TFLOP/s",
                        "frac": net_tflops / tf_sus, "ms": net_ms},
        "mask": {"ms": mask_ms},
    }
    # per-kernel-class launch time per frame (region 3)
    kernels = {name: {"ms_per_frame": v[0] / k, "launches_per_frame": v[2] / k} for name, v in kern.items() if v[2]}
    conv_ms, conv_flops, conv_n = kern["conv"]
    conv_tf = conv_flops / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else 0.0
    kernels["conv"].update(bound="tensor", achieved=conv_tf, peak=tf_sus, unit="TFLOP/s", frac=conv_tf / tf_sus,
                           flops_per_launch=conv_flops / max(conv_n, 1))
    m_ms = sum(kern[c][0] for c in ("march_main", "march_shadow", "march_composite"))
    m_gbs = (samples_per_frame * BYTES_PER_SAMPLE + rays_per_frame * 20) * k / (m_ms / 1e3) / 1e9 if m_ms > 0 else 0.0
    marcher = {"bound": "hbm", "achieved": m_gbs, "peak": hbm, "unit": "GB/s", "frac": m_gbs / hbm,
               "ms_per_frame": m_ms / k}
    # dominant kernel = the class with the most launch time per frame: the tcgen05 conv engine
    # (every D/K conv of the W-Net) or the three wavefront marcher passes taken together
    dom = "conv" if conv_ms >= m_ms else "marcher"
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(dom, {}).get("dram_bytes_per_launch")
    if dom == "conv":
        roof = {"bound": "tensor", "achieved": conv_tf, "peak": tf_sus, "unit": "TFLOP/s", "frac": conv_tf / tf_sus,
                "traffic": traffic, "kernel": "conv3x3_tc_kernel (all W-Net convs of a frame)",
                "launches_per_frame": conv_n / k,
                "how": "sum of algorithmic conv FLOPs / sum of launch durations (CUDA events per launch)",
                "peak_source": f"{src} ({peak_kind})", "frac_vs_sustained": conv_tf / tf_sus_raw}
    else:
        roof = dict(marcher, traffic=traffic, kernel="march_wave_{main,shadow,composite}_kernel",
                    how=f"({BYTES_PER_SAMPLE} B/sample + 20 B/ray) / summed launch durations",
                    peak_source=f"{src} (copy bandwidth)")
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sec, desc, threads = cpu_frame_sample(cfg, frames=2)
        cpu = {"value": 1.0 / sec, "unit": "frames/s", "cores": threads, "kind": "port", "sample": desc}
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": k, "warmup": wu,
        "ms_per_step": elapsed_ms / k, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp16 net (fp32 acc) / fp32 march", "data": "synthetic",
        "config": {"workload": cfg["name"], "film": [w, h], "volume": [n, n, n], "path_frames": PATH_FRAMES,
                   "parallelism": f"independent frame streams x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (512 MiB volume, ~1.6 GB activations per frame)"},
        "gsamples_per_s": world * samples_per_frame * k / (elapsed_ms / 1e3) / 1e9,
        "samples_per_frame": samples_per_frame, "active_rays_per_frame": rays_per_frame,
        "phase_ms": {"mask": mask_ms, "march": march_ms, "reconstruct": net_ms},
        "timing": {"pipelined_ms_per_frame": pipe_ms / k, "serial_ms_per_frame": serial_ms / k,
                   "serial_fps": whole_job_rate(k, world, serial_ms / 1e3),
                   "how": "value = K frames through the frame loop (FramePipeline.run_pipelined -> the C ABI's "
                          "fv_frames: each frame one replayed CUDA graph -- frame t's network with frame t+1's "
                          "mask + march forked off it after its 6th conv (FV_MARCH_AHEAD) and frame t-1's K "
                          "filter chain + output stage after its 12th (FV_KCHAIN_SPLIT / FV_KCHAIN_AT), the "
                          "per-frame camera / fovea read from a device parameter block), CUDA events on the "
                          "pipeline stream; phase_ms from the same frames in serial order with events "
                          "between the phases"},
        "roofline": roof, "stages": stages, "kernels": kernels, "marcher": marcher,
        "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": h * w * 3 * 4, "serial_fv_frame_fps": e2e_serial_fps,
                "how": f"fv_frames C-ABI call over {ke} frames (run right after the headline region), wall "
                       "clock: per frame camera + fovea by value "
                       "(H2D through the device parameter block), (H,W,3) f32 image D2H into pinned host memory; "
                       "each image's copy overlaps the following frames' compute (copy stream)"},
        "gpu_launches": launches, "clocks": clk, "cpu_baseline": cpu, "device_memory_gb": device_memory_gb(),
        "sustained": sustained,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_strip_sample(cfg, vol, rows=256, frames=1):
    """cpu_baseline of the --shard line: the oracle on a full-width strip of `rows` rows through the
    fovea (its mask, the C fp64 march of its active rays, the fp32 network on the strip), scaled to
    the frame by rows; a whole 4K frame at 1024^3 would take minutes on the host."""
    from oracle import fovray_oracle as O

    h, w, n = cfg["height"], cfg["width"], cfg["vol"]
    r0 = (h // 2 - rows // 2) // 8 * 8
    stack = O.load_rnkstack(ROOT / "paper_2209_09965_b200" / "data" / "stbn_64x64x8_s1.noise")
    tau = O.tau_map(h, w, ((w - 1) / 2, (h - 1) / 2), cfg["sigma"], cfg["pb"], O.pixel_scale_for_film(h, w))
    params = O.init_params(O.FULL_BLOCKS, 0, fp16_weights=True)
    state = None
    secs = []
    for i in range(frames):
        t0 = time.perf_counter()
        bits = O.sample_mask(stack, h, w, i, tau)[r0:r0 + rows]
        pix = O.compact(bits) + r0 * w
        pos, look = O.orbit_camera(i, PATH_FRAMES, (n, n, n))
        rgba, _ = O.render(vol, (1, 1, 1), O.DEFAULT_LUT, ("dir", (-1.0, -1.0, -0.5), (1, 1, 1)),
                           dict(position=pos, look_at=look, fov_y=45.0, width=w, height=h), pix=pix)
        img = np.zeros((rows * w, 4), np.float32)
        img[pix - r0 * w] = rgba
        m = bits.astype(np.float32)
        x = np.concatenate([np.moveaxis(img.reshape(rows, w, 4), -1, 0) * m[None], m[None]], 0)
        _, _, state = O.net_forward(params, O.FULL_BLOCKS, x, state)
        secs.append((time.perf_counter() - t0) * h / rows)
    desc = (f"{frames} frame(s) of a {w}x{rows} strip through the fovea (rows {r0}..{r0 + rows}): oracle mask, C fp64 "
            f"march of the strip's active rays on all {len(os.sched_getaffinity(0))} host threads, fp32 NumPy/BLAS "
            f"FULL_BLOCKS net on the strip; per-frame time scaled by {h}/{rows} rows; CPU {cpu_model()}")
    return float(np.mean(secs)), desc, len(os.sched_getaffinity(0))


def run_sharded(args, cfg):
    """One frame stream split across the ranks (config 5: --config c5 --shard): every rank marches
    its 32-ray packets of each frame, one all_gather_into_tensor of 12-byte records gives every
    rank the frame's rays, and each rank reconstructs its row strip on a window (strip + halo),
    exchanging the recurrent boundary bands with its neighbours after the frame
    (sharded.StripShardedPipeline; --shard-replicated: the round-1 replicated network). Strong
    scaling: the job renders K frames whatever N is; time = max over ranks."""
    import torch

    rank, world, local = dist_env()
    tdev = init_rank_device(local, world)
    group = None
    from paper_2209_09965_b200 import _lib
    from paper_2209_09965_b200 import network as N
    from paper_2209_09965_b200.noise import default_stack
    from paper_2209_09965_b200.renderer import OrbitPathSpec, RenderSettings, orbit_cameras
    from paper_2209_09965_b200.sample_maps import FoveaConfig, pixel_scale_for_film
    from paper_2209_09965_b200.sharded import ShardedFramePipeline, StripShardedPipeline
    from paper_2209_09965_b200.throughput import default_scene

    h, w, n = cfg["height"], cfg["width"], cfg["vol"]
    scene = default_scene("sphere_shells", (n, n, n))
    net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.FULL_BLOCKS), seed=0), "fp16")
    cams = orbit_cameras(OrbitPathSpec(n_frames=PATH_FRAMES), scene.volume, w, h)
    fovea = FoveaConfig(focus=((w - 1) / 2.0, (h - 1) / 2.0), sigma=cfg["sigma"], base_density=cfg["pb"],
                        pixel_scale=pixel_scale_for_film((h, w)))
    strip = not args.shard_replicated
    cls = StripShardedPipeline if strip else ShardedFramePipeline
    pipe = cls(scene, net, (h, w), default_stack(), RenderSettings(), rank=rank, world=world, group=group)
    ctx = pipe.pipe.ctx
    k, wu = args.steps, args.warmup
    clocks = ClockSampler(local, ROOT / "gpurun_out" / f"clocks_r{rank}.csv") if rank == 0 else None
    for j in range(wu):
        pipe.step(cams[j % PATH_FRAMES], fovea, j)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches()
    ctx.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j in range(wu, wu + k):  # the same frames on every rank: each marches its share
        pipe.step(cams[j % PATH_FRAMES], fovea, j)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world, device=tdev)
    launches = ctx.launches() - l0
    st = ctx.stats()
    # the conv roofline of this rank's network over the same frames, kernel timing on
    ctx.set_kernel_timing(True)
    for j in range(wu, wu + min(k, 4)):
        pipe.step(cams[j % PATH_FRAMES], fovea, j)
    torch.cuda.synchronize()
    conv_ms, conv_flop, conv_n = ctx.kernel_time(_lib.KERNEL_CLASSES["conv"])
    ctx.set_kernel_timing(False)
    # end to end: every rank copies its part of each frame's image to pinned host memory (its owned
    # strip; the replicated design: rank 0 the whole image); wall clock, max over ranks
    part = pipe.owned_rgb(rank) if strip else pipe.rgb
    host = torch.empty(tuple(part.shape), dtype=torch.float32).pin_memory()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for j in range(wu + k, wu + 2 * k):
        pipe.step(cams[j % PATH_FRAMES], fovea, j)
        if strip or rank == 0:
            host.copy_(pipe.owned_rgb(rank) if strip else pipe.rgb, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, world, device=tdev)
    clk = clocks.stop() if clocks else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, desc, thr = cpu_strip_sample(cfg, scene.volume.data)
        cpu = {"value": 1.0 / sec, "unit": "frames/s", "cores": thr, "kind": "port", "sample": desc}
    if rank == 0:
        hbm, tf_burst, tf_sus, src = load_peaks()
        at_max = bool(clk and clk.get("sm_mhz") and clk["sm_mhz"] >= 0.95 * clk.get("sm_max_mhz", 1e9))
        peak = tf_burst if at_max else tf_sus
        conv_tf = conv_flop / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else 0.0
        samples = (st.samples_main + st.samples_shadow) / k  # this rank's share
        geo = getattr(pipe, "geo", None)
        line = {
            "metric": METRIC, "value": k / (ms / 1e3), "unit": "frames/s", "n_gpus": world, "steps": k,
            "warmup": wu, "ms_per_step": ms / k, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp16 net (fp32 acc) / fp32 march", "data": "synthetic",
            "config": {"workload": cfg["name"], "film": [w, h], "volume": [n, n, n], "path_frames": PATH_FRAMES,
                       "parallelism": (f"one frame stream over {world} GPUs: march in 32-ray packets, record "
                                       "all_gather_into_tensor (NCCL), reconstruction in row strips on windows of "
                                       f"strip + {pipe.halo} rows with a per-frame band exchange" if strip else
                                       f"one frame stream, march sharded in 32-ray packets over {world} GPUs, "
                                       "record all-gather (NCCL), replicated reconstruction"),
                       "strips": geo, "l2": "inputs larger than L2"},
            "samples_per_frame_rank0": samples,
            "record_gather": ({"records_per_rank": pipe.frame_capacity(), "pixel_bound": pipe.cap,
                               "bytes_per_frame": world * pipe.frame_capacity() * 12,
                               "how": "sized per frame by the compacted ray count (last frame shown)"}
                              if strip else None),
            "e2e": {"value": k / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": int(host.numel() * 4),
                    "how": "pipe.step per frame + pinned D2H of the rank's part of the image, wall clock"},
            "gpu_launches": launches, "clocks": clk, "device_memory_gb": device_memory_gb(),
            "roofline": {"bound": "tensor", "achieved": conv_tf, "peak": peak, "unit": "TFLOP/s",
                         "frac": conv_tf / peak, "traffic": None,
                         "kernel": "conv3x3_tc_kernel (all W-Net convs of rank 0's window)",
                         "launches_per_frame": conv_n / min(k, 4),
                         "how": "algorithmic conv FLOPs of the window / summed launch durations (CUDA events)",
                         "peak_source": f"{src} ({'burst' if at_max else 'sustained'} dense fp16/bf16)"},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sustained", action="store_true", help="skip the ~1 s sustained-clock run")
    ap.add_argument("--shard", action="store_true",
                    help="split each frame across the ranks (config 5: march by packets, network by row strips) "
                         "instead of independent frame streams")
    ap.add_argument("--shard-replicated", action="store_true",
                    help="with --shard: the round-1 design (march split, network replicated on every rank)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.shard:
        run_sharded(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
