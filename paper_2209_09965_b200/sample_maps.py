"""Foveated sample maps: tau thresholds, binary masks and compaction, on the GPU.

Drop-in for the reference's pkg/src/fovray/sample_maps.py. The three calls the
per-frame loop makes -- build_tau_map (:89-105), build_sample_mask (:128-132) and
compact_mask (:161-171) -- run as ONE fused CUDA kernel (fv_mask_compact): fp64
tau, the noise-stack comparison and a decoupled look-back row-major scan that
writes the compacted index list. The host objects below keep the reference's
types and validation; their arrays live on the device and are copied to NumPy
only when a caller reads them.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .noise import NoiseStack

DEFAULT_PIXEL_SCALE = 1.0 / 32.0
FAST_PRESET = {"base_density": 0.03, "sigma": 0.02}
HIFI_PRESET = {"base_density": 0.07, "sigma": 0.06}


def pixel_scale_for_film(dims: tuple[int, int], fraction: float = 0.45) -> float:
    """Offset scale keeping the fovea a fixed fraction of the film (sample_maps.py:31-40)."""
    h, w = dims
    return float(np.sqrt(2.0 / FAST_PRESET["sigma"]) / (fraction * min(h, w)))


@dataclass(frozen=True)
class FoveaConfig:
    """Focal point plus fall-off parameters (sample_maps.py:43-59)."""

    focus: tuple[float, float]
    sigma: float = 0.02
    base_density: float | np.ndarray = 0.03
    pixel_scale: float = DEFAULT_PIXEL_SCALE

    def __post_init__(self):
        if self.sigma < 0:
            raise ValueError(f"sigma must be >= 0, got {self.sigma}")
        if not np.all(np.isfinite(self.focus)):
            raise ValueError("focus must be finite")
        pb = np.asarray(self.base_density)
        if pb.min() < 0.0 or pb.max() > 1.0:
            raise ValueError("base density must lie in [0,1]")

    def c_struct(self) -> _lib.FvFovea:
        f = _lib.FvFovea()
        f.focus[0], f.focus[1] = float(self.focus[0]), float(self.focus[1])
        f.sigma = float(self.sigma)
        pb = np.asarray(self.base_density)
        f.base_density = float(pb) if pb.ndim == 0 else 0.0
        f.pixel_scale = float(self.pixel_scale)
        return f


def foveal_density(offset, sigma: float, pixel_scale: float = DEFAULT_PIXEL_SCALE):
    """exp(-0.5*((dx*s)^2+(dy*s)^2)*sigma) (sample_maps.py:62-68) over broadcast pixel offsets,
    evaluated by fv_foveal_density with the mask kernel's fp64 arithmetic."""
    import torch

    dx, dy = np.broadcast_arrays(np.asarray(offset[0], dtype=np.float64), np.asarray(offset[1], dtype=np.float64))
    shape = dx.shape
    tx = torch.as_tensor(np.ascontiguousarray(dx).reshape(-1), device="cuda")
    ty = torch.as_tensor(np.ascontiguousarray(dy).reshape(-1), device="cuda")
    out = torch.empty_like(tx)
    ctx = _lib.context()
    _lib.check(ctx.lib.fv_foveal_density(ctx.h, _lib.ptr(tx), _lib.ptr(ty), int(tx.numel()), float(sigma),
                                         float(pixel_scale), _lib.ptr(out)))
    res = out.cpu().numpy().reshape(shape)
    return float(res) if res.ndim == 0 else res


class TauMap:
    """Per-pixel threshold field (sample_maps.py:71-86).

    Built from a FoveaConfig it is lazy: the fused mask kernel evaluates tau inline
    and `values` materialises the fp64 map on demand. Built from explicit values it
    is uploaded once and thresholded as given.
    """

    def __init__(self, values=None, *, cfg: FoveaConfig | None = None,
                 dims: tuple[int, int] | None = None):
        self.cfg = cfg
        self._dev = None
        self._host = None
        self._pb_dev = None
        if values is not None:
            v = np.asarray(values, dtype=np.float64)
            if v.ndim != 2:
                raise ValueError(f"tau map must be 2D, got shape {v.shape}")
            if v.min() < 0.0 or v.max() > 1.0:
                raise ValueError("tau values must lie in [0,1]")
            v = v.copy()
            v.setflags(write=False)
            self._host = v
            self._dims = v.shape
        else:
            self._dims = tuple(dims)

    @property
    def dims(self) -> tuple[int, int]:
        return tuple(self._dims)

    def pb_map_dev(self):
        pb = np.asarray(self.cfg.base_density, dtype=np.float64)
        if pb.ndim != 2:
            return None
        if self._pb_dev is None:
            import torch

            self._pb_dev = torch.as_tensor(np.ascontiguousarray(pb), device="cuda")
        return self._pb_dev

    def values_dev(self):
        import torch

        if self._dev is None:
            if self._host is not None:
                self._dev = torch.as_tensor(np.array(self._host), device="cuda")  # writable copy
            else:
                ctx = _lib.context()
                h, w = self.dims
                t = torch.empty((h, w), dtype=torch.float64, device="cuda")
                f = self.cfg.c_struct()
                _lib.check(ctx.lib.fv_tau_map(ctx.h, h, w, C.byref(f), _lib.ptr(self.pb_map_dev()),
                                              _lib.ptr(t)))
                self._dev = t
        return self._dev

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            v = self.values_dev().cpu().numpy()
            v.setflags(write=False)
            self._host = v
        return self._host


def build_tau_map(cfg: FoveaConfig, dims: tuple[int, int]) -> TauMap:
    """tau = P_f + (1 - P_f) * P_b over an (H, W) grid (sample_maps.py:89-105)."""
    h, w = dims
    if h < 1 or w < 1:
        raise ValueError(f"dims must be positive, got {dims}")
    pb = np.asarray(cfg.base_density, dtype=np.float64)
    if pb.ndim == 2 and pb.shape != (h, w):
        raise ValueError(f"per-pixel base density shape {pb.shape} != dims {(h, w)}")
    return TauMap(cfg=cfg, dims=(h, w))


class SampleMask:
    """Binary decision per pixel for one frame (sample_maps.py:108-125); bits live on the GPU."""

    def __init__(self, bits=None, frame: int = 0, *, bits_dev=None, compact=None):
        import torch

        self.frame = frame
        self._compact = compact
        if bits_dev is not None:
            self._dev = bits_dev
            self._host = None
        else:
            b = np.asarray(bits)
            if b.ndim != 2 or b.dtype != np.bool_:
                raise ValueError("mask bits must be a 2D bool array")
            b = b.copy()
            self._dev = torch.as_tensor(b.view(np.uint8), device="cuda")
            b.setflags(write=False)
            self._host = b

    @property
    def dims(self) -> tuple[int, int]:
        return tuple(self._dev.shape)

    @property
    def bits_dev(self):
        """(H, W) uint8 CUDA tensor."""
        return self._dev

    @property
    def bits(self) -> np.ndarray:
        if self._host is None:
            b = self._dev.cpu().numpy().astype(bool)
            b.setflags(write=False)
            self._host = b
        return self._host

    def density(self) -> float:
        """Fraction of set bits: exact count / pixels in fp64, as numpy's bool mean."""
        return int(self._dev.sum(dtype=__import__("torch").int64).item()) / self._dev.numel()


def build_sample_mask(noise: NoiseStack, frame: int, tau: TauMap) -> SampleMask:
    """M(u,v) = 1 iff N(u,v) < tau(u,v) with toroidal noise (sample_maps.py:128-132).

    One fused launch also produces the compacted list (returned by compact_mask).
    """
    import torch

    ctx = _lib.context()
    ctx.ensure_noise(noise)
    h, w = tau.dims
    bits = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    idx = torch.empty((h * w,), dtype=torch.int32, device="cuda")
    k = torch.empty((1,), dtype=torch.int32, device="cuda")
    if tau.cfg is not None and tau._host is None:
        f = tau.cfg.c_struct()
        _lib.check(ctx.lib.fv_mask_compact(ctx.h, int(frame), h, w, C.byref(f),
                                           _lib.ptr(tau.pb_map_dev()), _lib.ptr(bits),
                                           _lib.ptr(idx), _lib.ptr(k), None))
    else:
        _lib.check(ctx.lib.fv_mask_compact_tau(ctx.h, int(frame), h, w, _lib.ptr(tau.values_dev()),
                                               _lib.ptr(bits), _lib.ptr(idx), _lib.ptr(k), None))
    comp = CompactIndexList(dims=(h, w), idx_dev=idx, k_dev=k)
    return SampleMask(frame=frame, bits_dev=bits, compact=comp)


def c_max(tau: TauMap) -> float:
    """Mean of tau over the frame: the ideal work fraction (sample_maps.py:135-137), a deterministic
    fp64 device sum (fv_tau_sum; tau evaluated inline unless the map holds explicit values)."""
    import torch

    ctx = _lib.context()
    h, w = tau.dims
    out = torch.empty((1,), dtype=torch.float64, device="cuda")
    if tau.cfg is not None and tau._host is None and tau._dev is None:
        f = tau.cfg.c_struct()
        _lib.check(ctx.lib.fv_tau_sum(ctx.h, h, w, C.byref(f), _lib.ptr(tau.pb_map_dev()), None, _lib.ptr(out)))
    else:
        _lib.check(ctx.lib.fv_tau_sum(ctx.h, h, w, None, None, _lib.ptr(tau.values_dev()), _lib.ptr(out)))
    return float(out.item()) / (h * w)


class CompactIndexList:
    """Set pixels packed densely in row-major order (sample_maps.py:140-158).

    On the device the list is int32 flat indices v*W+u plus a device-side count; the
    reference's (k, 2) int64 (u, v) coords are produced on first access.
    """

    def __init__(self, coords=None, dims: tuple[int, int] = (0, 0), *, idx_dev=None, k_dev=None):
        import torch

        self.dims = tuple(dims)
        self._coords = None
        self._k = None
        if idx_dev is not None:
            self._idx = idx_dev
            self._kdev = k_dev
        else:
            c = np.asarray(coords)
            if c.ndim != 2 or c.shape[1] != 2:
                raise ValueError("coords must have shape (k, 2)")
            flat = c[:, 1].astype(np.int64) * self.dims[1] + c[:, 0]
            if np.any(np.diff(flat) <= 0):
                raise ValueError("coords must be strictly ascending in row-major order")
            c = c.astype(np.int64).copy()
            c.setflags(write=False)
            self._coords = c
            self._k = int(c.shape[0])
            self._idx = torch.as_tensor(flat.astype(np.int32), device="cuda")
            if self._idx.numel() == 0:
                self._idx = torch.zeros((1,), dtype=torch.int32, device="cuda")
            self._kdev = torch.tensor([self._k], dtype=torch.int32, device="cuda")

    @property
    def idx_dev(self):
        return self._idx

    @property
    def k_dev(self):
        return self._kdev

    @property
    def count(self) -> int:
        if self._k is None:
            self._k = int(self._kdev.item())
        return self._k

    @property
    def coords(self) -> np.ndarray:
        if self._coords is None:
            flat = self._idx[: self.count].cpu().numpy().astype(np.int64)
            w = self.dims[1]
            c = np.stack([flat % w, flat // w], axis=1)
            c.setflags(write=False)
            self._coords = c
        return self._coords


def compact_mask(mask: SampleMask) -> CompactIndexList:
    """Pack set bits in row-major order (sample_maps.py:161-171)."""
    if mask._compact is not None:
        return mask._compact
    import torch

    flat = torch.nonzero(mask.bits_dev.reshape(-1), as_tuple=False).reshape(-1).to(torch.int32)
    k = torch.tensor([flat.numel()], dtype=torch.int32, device="cuda")
    if flat.numel() == 0:
        flat = torch.zeros((1,), dtype=torch.int32, device="cuda")
    mask._compact = CompactIndexList(dims=mask.dims, idx_dev=flat, k_dev=k)
    return mask._compact


def scatter(compact: CompactIndexList, frame: int = 0) -> SampleMask:
    """Inverse of compact_mask (sample_maps.py:174-178)."""
    import torch

    h, w = compact.dims
    bits = torch.zeros((h * w,), dtype=torch.uint8, device="cuda")
    k = compact.count
    if k:
        bits[compact.idx_dev[:k].long()] = 1
    return SampleMask(frame=frame, bits_dev=bits.reshape(h, w), compact=compact)


def draw_direct_samples(cfg: FoveaConfig, noise_frame, count: int, rng: np.random.Generator) -> np.ndarray:
    """Stochastic pixel positions with probability proportional to tau (sample_maps.py:181-198).

    Inverse-CDF sampling over the fp64 tau map on the device (fv_direct_draws: tau, the cumulative
    sum, the normalisation and the right-sided binary search); the uniforms come from the caller's
    NumPy generator, so the draws follow the reference's random stream. Duplicates are expected:
    that is direct sampling's documented weakness versus compaction. Returns (count, 2) int64 (u, v)."""
    idx = direct_draws_dev(cfg, np.asarray(noise_frame).shape, count, rng)
    w = np.asarray(noise_frame).shape[1]
    flat = idx.cpu().numpy().astype(np.int64)
    return np.stack([flat % w, flat // w], axis=1)


def direct_draws_dev(cfg: FoveaConfig, dims: tuple[int, int], count: int, rng: np.random.Generator):
    """The draws of draw_direct_samples as a (count,) int32 CUDA tensor of flat indices v*W+u."""
    import torch

    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    h, w = dims
    r = torch.as_tensor(rng.random(count), device="cuda")
    idx = torch.empty((count,), dtype=torch.int32, device="cuda")
    tau = build_tau_map(cfg, (h, w))
    ctx = _lib.context()
    f = cfg.c_struct()
    _lib.check(ctx.lib.fv_direct_draws(ctx.h, h, w, C.byref(f), _lib.ptr(tau.pb_map_dev()), None, _lib.ptr(r),
                                       int(count), _lib.ptr(idx)))
    return idx


def cmax_sweep_rows(settings: list[tuple[float, float]], noise: NoiseStack, dims: tuple[int, int],
                    focus: tuple[float, float] | None = None) -> list[tuple]:
    """(P_b, sigma, c_max, measured_density) rows over the noise loop (sample_maps.py:209-223); the
    masks come from the fused mask kernel."""
    h, w = dims
    if focus is None:
        focus = ((w - 1) / 2.0, (h - 1) / 2.0)
    rows = []
    for pb, sigma in settings:
        cfg = FoveaConfig(focus=focus, sigma=sigma, base_density=pb)
        tau = build_tau_map(cfg, dims)
        dens = np.mean([build_sample_mask(noise, f, tau).density() for f in range(noise.frames)])
        rows.append((pb, sigma, c_max(tau), float(dens)))
    return rows
