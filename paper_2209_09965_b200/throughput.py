"""Per-frame throughput driver: the device twin of bench.cmd_bench_throughput.

Mirrors pkg/src/fovray/bench.py:57-88 (ExperimentSpec, default_scene), :166-175
(_reconstruct_frame) and :178-222 (cmd_bench_throughput) with the same CSV
schema `frame,mask_ms,render_ms,reconstruct_ms,total_ms`; phase times are CUDA
event intervals of the FramePipeline instead of host wall-clock.
"""
from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .network import WNetParams, load_network, quantized_net
from .noise import NoiseStack, default_stack
from .pipeline import FramePipeline
from .renderer import OrbitPathSpec, RenderSettings, Scene, orbit_cameras, render_full, render_sparse_compact
from .sample_maps import FAST_PRESET, HIFI_PRESET, FoveaConfig, pixel_scale_for_film
from .volume import Camera, Light, TransferFunction, make_procedural_volume

DATASETS = ("sphere_shells", "vortex_field", "box_lattice")
MODES = ("ovr", "fast", "hifi")


@dataclass(frozen=True)
class ExperimentSpec:
    dataset: str = "sphere_shells"
    mode: str = "ovr"
    frames: int = 16
    seed: int = 0
    width: int = 320
    height: int = 180
    out_dir: str | Path = "bench_out"
    volume_dims: tuple[int, int, int] = (32, 32, 32)

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.dataset not in DATASETS:
            raise ValueError(f"dataset must be one of {DATASETS}, got {self.dataset!r}")

    def fovea(self) -> FoveaConfig | None:
        if self.mode == "ovr":
            return None
        preset = FAST_PRESET if self.mode == "fast" else HIFI_PRESET
        return FoveaConfig(focus=((self.width - 1) / 2.0, (self.height - 1) / 2.0), sigma=preset["sigma"],
                           base_density=preset["base_density"],
                           pixel_scale=pixel_scale_for_film((self.height, self.width)))


def default_scene(dataset: str, dims: tuple[int, int, int] = (32, 32, 32)) -> Scene:
    """bench.default_scene (bench.py:85-88): procedural volume, default TF, light (-1,-1,-0.5)."""
    vol = make_procedural_volume(dataset, dims)
    return Scene(volume=vol, tf=TransferFunction.default(),
                 light=Light(direction=(-1.0, -1.0, -0.5), intensity=(1.0, 1.0, 1.0)))


def _reconstruct_frame(net: WNetParams, sparse_rgba, mask_bits, state):
    """x = rgba*m (++ m), forward_full, clip to [0,1] (bench.py:166-175); returns (img (H,W,3), state').

    With the mask channel the packing and the clip run on the device (fv_pack_input, the output
    stage); without it the rgba*m product is formed on the device and fed to forward_full."""
    import torch

    from .network import forward_full, forward_sparse

    rgba = torch.as_tensor(np.asarray(getattr(sparse_rgba, "rgba", sparse_rgba), dtype=np.float32)
                           if not isinstance(sparse_rgba, torch.Tensor) else sparse_rgba, device="cuda")
    mb = torch.as_tensor(np.asarray(mask_bits) if not isinstance(mask_bits, torch.Tensor) else mask_bits,
                         device="cuda")
    if net.config.include_mask_channel:
        rgb, _, _, state = forward_sparse(net, rgba, mb.to(torch.uint8), state)
        return rgb.cpu().numpy(), state
    x = rgba.permute(2, 0, 1)[None] * mb.to(torch.float32)[None, None]
    o, _, state = forward_full(net, x, state)
    return torch.clamp(o.dev[0].permute(1, 2, 0), 0.0, 1.0).cpu().numpy(), state


def _write_csv(path: Path, header, rows, echo: dict) -> None:
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="") as f:
        f.write("# " + json.dumps(echo) + "\n")
        w = csv.writer(f)
        w.writerow(header)
        w.writerows(rows)


def cmd_bench_throughput(spec: ExperimentSpec, checkpoint=None, noise: NoiseStack | None = None,
                         settings: RenderSettings = RenderSettings(), write: bool = True) -> list[tuple]:
    """Fly-through timing rows per frame (bench.py:178-222), all phases on the GPU."""
    import torch

    net = None
    if spec.mode != "ovr":
        if checkpoint is None:
            raise ValueError(f"mode {spec.mode!r} needs a trained checkpoint")
        net = checkpoint if isinstance(checkpoint, WNetParams) else load_network(checkpoint)[0]
    scene = default_scene(spec.dataset, spec.volume_dims)
    cams = orbit_cameras(OrbitPathSpec(n_frames=spec.frames), scene.volume, spec.width, spec.height)
    noise = noise if noise is not None else default_stack()
    fovea = spec.fovea()
    pipe = FramePipeline(scene, net, (spec.height, spec.width), noise, settings)
    rows = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i, cam in enumerate(cams):
        if spec.mode == "ovr":
            e0.record(pipe.ctx.stream)
            pipe.dense(cam)
            e1.record(pipe.ctx.stream)
            e1.synchronize()
            mask_ms, render_ms, rec_ms = 0.0, e0.elapsed_time(e1), 0.0
        else:
            mask_ms, render_ms, rec_ms = pipe.step(cam, fovea, i, timed=True)
        rows.append((i, mask_ms, render_ms, rec_ms, mask_ms + render_ms + rec_ms))
    if write:
        echo = {"dataset": spec.dataset, "mode": spec.mode, "frames": spec.frames,
                "film": [spec.width, spec.height], "seed": spec.seed, "device": "cuda",
                "preset": None if fovea is None else
                {"p_b": float(np.asarray(fovea.base_density)), "sigma": fovea.sigma}}
        out = Path(spec.out_dir) / "throughput"
        _write_csv(out / f"{spec.dataset}_{spec.mode}.csv",
                   ["frame", "mask_ms", "render_ms", "reconstruct_ms", "total_ms"], rows, echo)
        totals = [r[4] for r in rows]
        _write_csv(out / f"{spec.dataset}_{spec.mode}_summary.csv",
                   ["dataset", "mode", "mean_total_ms", "std_total_ms"],
                   [(spec.dataset, spec.mode, float(np.mean(totals)), float(np.std(totals)))], echo)
    return rows


def cmd_bench_cmax(taus=(0.01, 0.03, 0.05, 0.1, 0.2, 0.5, 1.0), dims: tuple[int, int] = (180, 320),
                   repeats: int = 3, dataset: str = "vortex_field", out_dir: str | Path | None = "bench_out",
                   volume_dims: tuple[int, int, int] = (48, 48, 48), seed: int = 0) -> list[tuple]:
    """Frame time vs uniform threshold for the naive and compacted renderers (bench.py:111-163).

    Film-sized uniform rank noise, so the work-item count is round(tau*H*W) up to rounding. Each
    render is timed on the device (CUDA events, median of warm repeats). Returns the CSV rows
    (tau, t_naive_ms, t_compact_ms, c_max, t_full_ms, work_items, mean_compact_ms, std_compact_ms);
    with out_dir, writes cmax/cmax_sweep.csv and cmax/cmax_settings.csv as the reference does.
    """
    from .noise import gen_uniform_noise
    from .renderer import render_sparse_naive
    from .sample_maps import TauMap, build_sample_mask, c_max, cmax_sweep_rows, compact_mask

    if min(taus) <= 0 or max(taus) > 1:
        raise ValueError("taus must lie in (0, 1]")
    h, w = dims
    scene = default_scene(dataset, volume_dims)
    center = scene.volume.center()
    diag = float(np.linalg.norm(scene.volume.extent))
    cam = Camera(position=tuple(center + diag * np.array([1.0, 0.7, 1.2])), look_at=tuple(center),
                 fov_y=40.0, width=w, height=h)
    noise = gen_uniform_noise(h, w, 2, seed=seed)
    settings = RenderSettings()
    render_full(scene, cam, settings)  # warm-up (brick cache, context)
    t_full = min(render_full(scene, cam, settings).render_ms for _ in range(repeats))
    rows = []
    for tau in taus:
        tmap = TauMap(values=np.full((h, w), float(tau)))
        mask = build_sample_mask(noise, 0, tmap)
        comp = compact_mask(mask)
        render_sparse_naive(scene, cam, mask, settings)
        render_sparse_compact(scene, cam, comp, settings)
        naive_ts = [render_sparse_naive(scene, cam, mask, settings).render_ms for _ in range(repeats)]
        compact_ts = [render_sparse_compact(scene, cam, comp, settings).render_ms for _ in range(repeats)]
        rows.append((tau, float(np.median(naive_ts)), float(np.median(compact_ts)), c_max(tmap), t_full,
                     comp.count, float(np.mean(compact_ts)), float(np.std(compact_ts))))
    if out_dir is not None:
        echo = {"taus": list(taus), "dims": list(dims), "repeats": repeats, "dataset": dataset,
                "volume_dims": list(volume_dims), "seed": seed, "device": "cuda",
                "timing": "median of warm repeats, CUDA events around each render, ms"}
        out = Path(out_dir) / "cmax"
        _write_csv(out / "cmax_sweep.csv",
                   ["tau", "t_naive_ms", "t_compact_ms", "c_max", "t_full_ms", "work_items",
                    "mean_compact_ms", "std_compact_ms"], rows, echo)
        settings_rows = cmax_sweep_rows(
            [(FAST_PRESET["base_density"], FAST_PRESET["sigma"]),
             (HIFI_PRESET["base_density"], HIFI_PRESET["sigma"]), (0.01, 0.02), (0.10, 0.02)],
            default_stack(), dims)
        _write_csv(out / "cmax_settings.csv", ["p_b", "sigma", "c_max", "measured_density"], settings_rows, echo)
    return rows


_quantized_net = quantized_net
