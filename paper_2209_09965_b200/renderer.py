"""Ray-marched volume rendering on the GPU: dense frames and compacted sparse frames.

Drop-in for the hot-path half of pkg/src/fovray/renderer.py. render_full
(:211-222) and render_sparse_compact (:262-288) call the CUDA marcher
(fv_render_full / fv_render_sparse) which follows _march (:150-195) and
shadow_transmittance (:109-147): front-to-back emission-absorption with opacity
correction 1-(1-a)^(dt/reference_step), depth at the first alpha>=0.5 crossing,
early termination and one shadow ray toward the light per contributing sample.
Frames keep their RGBA/depth on the device; `.rgba` / `.depth` copy to NumPy on
first access. Camera paths (orbit_cameras, :317-361) are host math.
"""
from __future__ import annotations

import ctypes as C
import csv
import json
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .sample_maps import CompactIndexList, SampleMask
from .volume import Camera, Light, TransferFunction, VolumeGrid


@dataclass(frozen=True)
class Scene:
    volume: VolumeGrid
    tf: TransferFunction
    light: Light | None = None


@dataclass(frozen=True)
class RenderSettings:
    """renderer.RenderSettings (renderer.py:44-65) + the device arithmetic tier.

    precision="fp32" marches in float (the fast tier: hardware-filtered samples); "fp32-strict" in
    float with software trilinear everywhere (the strict tier); "fp64" runs the per-sample
    arithmetic in double. Step control and sample positions are fp64 in all three.
    """

    step_size: float | None = None
    shadow_step_factor: float = 4.0
    early_term_alpha: float = 0.99
    background: tuple[float, float, float, float] = (0.0, 0.0, 0.0, 0.0)
    ambient: float = 0.25
    reference_step: float | None = None
    shadow_min_transmittance: float = 1e-3
    precision: str = "fp32"

    def __post_init__(self):
        if self.step_size is not None and self.step_size <= 0:
            raise ValueError("step_size must be > 0")
        if self.shadow_step_factor < 1:
            raise ValueError("shadow_step_factor must be >= 1")
        if self.precision not in ("fp32", "fp32-strict", "fp64"):
            raise ValueError(f"precision must be 'fp32', 'fp32-strict' or 'fp64', got {self.precision!r}")

    def resolve(self, vol: VolumeGrid) -> tuple[float, float]:
        base = float(min(vol.spacing))
        step = self.step_size if self.step_size is not None else 0.5 * base
        ref = self.reference_step if self.reference_step is not None else base
        return step, ref

    def c_struct(self) -> _lib.FvSettings:
        s = _lib.FvSettings()
        s.step_size = float(self.step_size) if self.step_size is not None else 0.0
        s.shadow_step_factor = float(self.shadow_step_factor)
        s.early_term_alpha = float(self.early_term_alpha)
        for i in range(4):
            s.background[i] = float(self.background[i])
        s.ambient = float(self.ambient)
        s.reference_step = float(self.reference_step) if self.reference_step is not None else 0.0
        s.shadow_min_transmittance = float(self.shadow_min_transmittance)
        s.precision = {"fp64": _lib.PREC_FP64, "fp32-strict": _lib.PREC_FP32_STRICT}.get(self.precision, _lib.PREC_FP32)
        return s


class Frame:
    """renderer.Frame (renderer.py:68-80) over device tensors.

    Nothing here synchronises the host at render time: the phase times are CUDA events read on first
    access of a `*_ms` field, the arrays copy to NumPy on first access of `.rgba` / `.depth`."""

    def __init__(self, rgba_dev, depth_dev=None, mask_ms=0.0, render_ms=0.0, reconstruct_ms=0.0,
                 total_ms=None, work_items=0, stats=None):
        self.rgba_dev = rgba_dev
        self.depth_dev = depth_dev
        self._ms = {"mask_ms": mask_ms, "render_ms": render_ms, "reconstruct_ms": reconstruct_ms,
                    "total_ms": total_ms}
        self._work = work_items
        self.stats = stats
        self._rgba = None
        self._depth = None

    def _get_ms(self, key):
        v = self._ms[key]
        if key == "total_ms" and v is None:
            return self.mask_ms + self.render_ms + self.reconstruct_ms
        if isinstance(v, tuple):  # (start, end) CUDA events: wait for the end on first access
            v[1].synchronize()
            v = float(v[0].elapsed_time(v[1]))
            self._ms[key] = v
        return v

    def _set_ms(self, key, v):
        self._ms[key] = v

    mask_ms = property(lambda self: self._get_ms("mask_ms"), lambda self, v: self._set_ms("mask_ms", v))
    render_ms = property(lambda self: self._get_ms("render_ms"), lambda self, v: self._set_ms("render_ms", v))
    reconstruct_ms = property(lambda self: self._get_ms("reconstruct_ms"),
                              lambda self, v: self._set_ms("reconstruct_ms", v))
    total_ms = property(lambda self: self._get_ms("total_ms"), lambda self, v: self._set_ms("total_ms", v))

    @property
    def work_items(self) -> int:
        if callable(self._work):
            self._work = int(self._work())
        return self._work

    @property
    def rgba(self) -> np.ndarray:
        if self._rgba is None:
            self._rgba = self.rgba_dev.cpu().numpy()
        return self._rgba

    @property
    def depth(self) -> np.ndarray | None:
        if self._depth is None and self.depth_dev is not None:
            self._depth = self.depth_dev.cpu().numpy()
        return self._depth

    @property
    def dims(self) -> tuple[int, int]:
        return int(self.rgba_dev.shape[0]), int(self.rgba_dev.shape[1])


class SparseFrame(Frame):
    def __init__(self, *args, mask=None, **kw):
        super().__init__(*args, **kw)
        self._mask = mask

    @property
    def mask(self) -> SampleMask | None:
        if callable(self._mask):
            self._mask = self._mask()
        return self._mask


def _light_ptr(scene: Scene):
    return C.byref(scene.light.c_struct()) if scene.light is not None else None


def render_full(scene: Scene, cam: Camera, settings: RenderSettings = RenderSettings(),
                stats: bool = False) -> Frame:
    """Dense baseline: one ray per pixel (renderer.py:211-222)."""
    import torch

    ctx = _lib.context()
    vol = scene.volume.handle(ctx, scene.tf)
    h, w = cam.height, cam.width
    rgba = torch.empty((h, w, 4), dtype=torch.float32, device="cuda")
    depth = torch.empty((h, w), dtype=torch.float32, device="cuda")
    st = _lib.FvStats() if stats else None
    camc, setc = cam.c_struct(), settings.c_struct()
    lightc = scene.light.c_struct() if scene.light is not None else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ctx.stream)
    _lib.check(ctx.lib.fv_render_full(ctx.h, vol, C.byref(camc), C.byref(lightc) if lightc else None,
                                      C.byref(setc), _lib.ptr(rgba), _lib.ptr(depth),
                                      C.byref(st) if st is not None else None))
    ev1.record(ctx.stream)
    return Frame(rgba, depth, render_ms=(ev0, ev1), work_items=w * h, stats=st)


def render_sparse_compact(scene: Scene, cam: Camera, compact: CompactIndexList,
                          settings: RenderSettings = RenderSettings(), stats: bool = False,
                          net_state=None, want_depth: bool = True) -> SparseFrame:
    """March exactly one work item per compacted entry and back-project (renderer.py:262-288).
    want_depth=False: no depth output (Frame.depth stays zero) -- the marcher then takes the
    frame loop's sample path (hardware-filtered main-pass samples, see csrc/march.cu)."""
    import torch

    if compact.dims != (cam.height, cam.width):
        raise ValueError(f"compact dims {compact.dims} != film {cam.height}x{cam.width}")
    if compact._coords is not None and compact.count and (
            compact._coords[:, 0].max() >= cam.width or compact._coords[:, 1].max() >= cam.height):
        raise ValueError("compact indices out of film range")
    ctx = _lib.context()
    vol = scene.volume.handle(ctx, scene.tf)
    h, w = cam.height, cam.width
    rgba = torch.zeros((h, w, 4), dtype=torch.float32, device="cuda")
    depth = torch.zeros((h, w), dtype=torch.float32, device="cuda")
    st = _lib.FvStats() if stats else None
    camc, setc = cam.c_struct(), settings.c_struct()
    lightc = scene.light.c_struct() if scene.light is not None else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ctx.stream)
    _lib.check(ctx.lib.fv_render_sparse(
        ctx.h, vol, C.byref(camc), C.byref(lightc) if lightc else None, C.byref(setc),
        _lib.ptr(compact.idx_dev), _lib.ptr(compact.k_dev), int(compact.idx_dev.numel()),
        _lib.ptr(rgba), _lib.ptr(depth) if want_depth else None, net_state, C.byref(st) if st is not None else None))
    ev1.record(ctx.stream)
    from .sample_maps import scatter

    return SparseFrame(rgba, depth, render_ms=(ev0, ev1), work_items=lambda: compact.count,
                       mask=lambda: scatter(compact), stats=st)


WARP_CHUNK = 64  # lanes per naive-mode execution group (renderer.py:34)


def render_sparse_naive(scene: Scene, cam: Camera, mask: SampleMask,
                        settings: RenderSettings = RenderSettings(), stats: bool = False) -> SparseFrame:
    """Thread-per-pixel march over every pixel of each occupied WARP_CHUNK-pixel chunk; lanes whose
    bit is clear idle and stay zero (renderer.py:225-259). Cost tracks occupied chunks, not set bits:
    the uncompacted baseline of the compression sweep."""
    import torch

    if mask.dims != (cam.height, cam.width):
        raise ValueError(f"mask dims {mask.dims} != film {cam.height}x{cam.width}")
    ctx = _lib.context()
    vol = scene.volume.handle(ctx, scene.tf)
    h, w = cam.height, cam.width
    rgba = torch.zeros((h, w, 4), dtype=torch.float32, device="cuda")
    depth = torch.zeros((h, w), dtype=torch.float32, device="cuda")
    idx = torch.empty((h * w,), dtype=torch.int32, device="cuda")
    k = torch.empty((1,), dtype=torch.int32, device="cuda")
    st = _lib.FvStats() if stats else None
    camc, setc = cam.c_struct(), settings.c_struct()
    lightc = scene.light.c_struct() if scene.light is not None else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ctx.stream)
    _lib.check(ctx.lib.fv_render_sparse_naive(
        ctx.h, vol, C.byref(camc), C.byref(lightc) if lightc else None, C.byref(setc),
        _lib.ptr(mask.bits_dev.contiguous()), _lib.ptr(idx), _lib.ptr(k), _lib.ptr(rgba), _lib.ptr(depth),
        C.byref(st) if st is not None else None))
    ev1.record(ctx.stream)
    return SparseFrame(rgba, depth, render_ms=(ev0, ev1), work_items=lambda: int(k.item()), mask=mask,
                       stats=st)


def render_sparse_direct(scene: Scene, cam: Camera, positions,
                         settings: RenderSettings = RenderSettings(), stats: bool = False) -> SparseFrame:
    """Render stochastically drawn (u, v) positions; duplicates are recomputed (renderer.py:291-314)."""
    import torch

    pos = np.asarray(positions, dtype=np.int64).reshape(-1, 2)
    h, w = cam.height, cam.width
    if pos.size and (pos[:, 0].min() < 0 or pos[:, 1].min() < 0 or pos[:, 0].max() >= w
                     or pos[:, 1].max() >= h):
        raise IndexError("direct sample positions out of film range")
    idx = torch.as_tensor((pos[:, 1] * w + pos[:, 0]).astype(np.int32), device="cuda")
    return _render_direct_idx(scene, cam, idx, settings, stats)


def _render_direct_idx(scene: Scene, cam: Camera, idx, settings: RenderSettings, stats: bool = False) -> SparseFrame:
    """render_sparse_direct over device flat indices v*W+u (in range; duplicates allowed)."""
    import torch

    ctx = _lib.context()
    vol = scene.volume.handle(ctx, scene.tf)
    h, w = cam.height, cam.width
    rgba = torch.zeros((h, w, 4), dtype=torch.float32, device="cuda")
    depth = torch.zeros((h, w), dtype=torch.float32, device="cuda")
    n = int(idx.numel())
    k = torch.tensor([n], dtype=torch.int32, device="cuda")
    st = _lib.FvStats() if stats else None
    camc, setc = cam.c_struct(), settings.c_struct()
    lightc = scene.light.c_struct() if scene.light is not None else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ctx.stream)
    if n:
        _lib.check(ctx.lib.fv_render_sparse(
            ctx.h, vol, C.byref(camc), C.byref(lightc) if lightc else None, C.byref(setc),
            _lib.ptr(idx), _lib.ptr(k), n, _lib.ptr(rgba), _lib.ptr(depth), None,
            C.byref(st) if st is not None else None))
    ev1.record(ctx.stream)

    def mask():
        bits = torch.zeros((h * w,), dtype=torch.uint8, device="cuda")
        if n:
            bits[idx.long()] = 1
        return SampleMask(bits=bits.reshape(h, w).cpu().numpy().astype(bool))

    return SparseFrame(rgba, depth, render_ms=(ev0, ev1), work_items=n, mask=mask, stats=st)


def render_flythrough(scene: Scene, cams: list[Camera], settings: RenderSettings = RenderSettings(),
                      mode: str = "full", noise=None, fovea=None, rng: np.random.Generator | None = None):
    """Render a camera path; returns (frames, timing rows) (renderer.py:385-432).

    Modes "full" (render_full), "naive", "compact" (mask + compaction, then the naive or compacted
    marcher) and "direct" (tau-proportional draws). Every frame is enqueued on the device without a
    host synchronisation (the noise frame index advances with the path frame); the timing rows
    (frame, mask_ms, render_ms, reconstruct_ms, total_ms) are CUDA-event intervals read once all
    frames are queued. ("direct" reads c_max back per frame: the draw count sizes the draws.)"""
    import torch

    from .sample_maps import build_sample_mask, build_tau_map, c_max, compact_mask, direct_draws_dev

    if not cams:
        raise ValueError("camera path must have at least one frame")
    if mode not in ("full", "naive", "compact", "direct"):
        raise ValueError(f"unknown flythrough mode {mode!r}")
    if mode != "full" and (noise is None or fovea is None):
        raise ValueError(f"mode {mode!r} needs a noise stack and a fovea config")
    rng = rng if rng is not None else np.random.default_rng(0)
    ctx = _lib.context()
    frames = []
    for i, cam in enumerate(cams):
        if mode == "full":
            fr = render_full(scene, cam, settings)
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            tau = build_tau_map(fovea, (cam.height, cam.width))
            if mode == "direct":
                count = max(1, int(round(c_max(tau) * cam.height * cam.width)))
                idx = direct_draws_dev(fovea, (cam.height, cam.width), count, rng)
            else:
                mask = build_sample_mask(noise, i, tau)
            e1.record(ctx.stream)
            if mode == "naive":
                fr = render_sparse_naive(scene, cam, mask, settings)
            elif mode == "compact":
                fr = render_sparse_compact(scene, cam, compact_mask(mask), settings)
            else:
                fr = _render_direct_idx(scene, cam, idx, settings)
            fr.mask_ms = (e0, e1)
        frames.append(fr)
    rows = [(i, fr.mask_ms, fr.render_ms, fr.reconstruct_ms, fr.total_ms) for i, fr in enumerate(frames)]
    return frames, rows


@dataclass(frozen=True)
class OrbitPathSpec:
    """Oscillating-zoom orbit around the volume centre (renderer.py:317-339)."""

    n_frames: int = 64
    radius_factor: float = 2.2
    zoom_amplitude: float = 0.35
    zoom_periods: float = 2.0
    yaw_turns: float = 1.0
    pitch_amplitude_deg: float = 25.0
    pitch_periods: float = 1.0
    speed_profile: str = "uniform"
    seed_phase: float = 0.0

    def parameter(self, i: int) -> float:
        if self.n_frames <= 1:
            return 0.0
        u = i / self.n_frames
        if self.speed_profile == "fast_slow_fast":
            return u + 0.22 * np.sin(2.0 * np.pi * u)
        return u


def orbit_cameras(spec: OrbitPathSpec, vol: VolumeGrid, width: int, height: int,
                  fov_y: float = 45.0) -> list[Camera]:
    """Camera path of renderer.orbit_cameras (renderer.py:342-361)."""
    center = vol.center()
    diag = float(np.linalg.norm(vol.extent))
    cams = []
    for i in range(spec.n_frames):
        s = spec.parameter(i)
        yaw = 2.0 * np.pi * (spec.yaw_turns * s + spec.seed_phase)
        pitch = np.deg2rad(spec.pitch_amplitude_deg) * np.sin(2.0 * np.pi * spec.pitch_periods * s)
        r = spec.radius_factor * diag * (1.0 + spec.zoom_amplitude *
                                         np.sin(2.0 * np.pi * spec.zoom_periods * s))
        pos = center + r * np.array([np.cos(pitch) * np.cos(yaw), np.sin(pitch),
                                     np.cos(pitch) * np.sin(yaw)])
        cams.append(Camera(position=tuple(pos), look_at=tuple(center), up=(0.0, 1.0, 0.0),
                           fov_y=fov_y, width=width, height=height))
    return cams


def save_camera_path(cams: list[Camera], path: str | Path, spec: OrbitPathSpec | None = None) -> None:
    doc = {"keyframes": [{"position": list(c.position), "look_at": list(c.look_at), "up": list(c.up),
                          "fov_y": c.fov_y, "width": c.width, "height": c.height} for c in cams]}
    if spec is not None:
        doc["generator"] = {k: getattr(spec, k) for k in spec.__dataclass_fields__}
    Path(path).write_text(json.dumps(doc, indent=1))


def load_camera_path(path: str | Path) -> list[Camera]:
    doc = json.loads(Path(path).read_text())
    return [Camera(position=tuple(k["position"]), look_at=tuple(k["look_at"]), up=tuple(k["up"]),
                   fov_y=k["fov_y"], width=k["width"], height=k["height"]) for k in doc["keyframes"]]


def write_timing_csv(path: str | Path, rows, config_echo: dict | None = None) -> None:
    with open(path, "w", newline="") as f:
        if config_echo:
            f.write("# " + json.dumps(config_echo) + "\n")
        writer = csv.writer(f)
        writer.writerow(["frame", "mask_ms", "render_ms", "reconstruct_ms", "total_ms"])
        writer.writerows(rows)
