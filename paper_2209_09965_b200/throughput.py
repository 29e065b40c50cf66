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
from .renderer import OrbitPathSpec, RenderSettings, Scene, orbit_cameras
from .sample_maps import FAST_PRESET, HIFI_PRESET, FoveaConfig, pixel_scale_for_film
from .volume import Light, TransferFunction, make_procedural_volume

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
    """x = rgba*m ++ m, forward_full, clip to [0,1] (bench.py:166-175); returns (img (H,W,3), state')."""
    import torch

    from .network import forward_full

    rgba = torch.as_tensor(np.asarray(getattr(sparse_rgba, "rgba", sparse_rgba), dtype=np.float32)
                           if not isinstance(sparse_rgba, torch.Tensor) else sparse_rgba, device="cuda")
    m = torch.as_tensor(np.asarray(mask_bits) if not isinstance(mask_bits, torch.Tensor) else mask_bits,
                        device="cuda").to(torch.float32)
    x = rgba.permute(2, 0, 1)[None] * m[None, None]
    if net.config.include_mask_channel:
        x = torch.cat([x, m[None, None]], dim=1)
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


_quantized_net = quantized_net
