"""Rank-noise stacks consumed by the foveated mask (lookup side only).

Mirrors the reference's NoiseStack / RNKSTACK cache (pkg/src/fovray/noise.py:31-57,
:432-468). Generating blue / spatio-temporal blue noise is an offline, sequential
process the reference caches to disk once; this package ships that cache for the
pipeline default (STBN 64x64x8, seed 1 -- `default_stack()` in noise.py:456-468)
and uploads it to the GPU, where the mask kernel performs the toroidal lookup
`stack[frame % T][v % H][u % W]` (noise.py:378-384).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

DEFAULT_TILE = 64
DEFAULT_FRAMES = 8
_CACHE_MAGIC = b"RNKSTACK"
_HEADER = "<8sIIIq dd"
_DATA = Path(__file__).resolve().parent / "data"


@dataclass(frozen=True)
class NoiseStack:
    """T x H x W stack of rank-noise values in [0,1) (noise.py:31-57)."""

    values: np.ndarray  # (T, H, W) float32
    seed: int = 0
    sigma_spatial: float = 0.0
    sigma_temporal: float = 0.0

    def __post_init__(self):
        v = np.asarray(self.values)
        if v.ndim != 3 or v.shape[0] < 1:
            raise ValueError(f"noise stack must be (T>=1, H, W), got {v.shape}")
        n = v.shape[1] * v.shape[2]
        ranks = ((np.arange(n) + 0.5) / n).astype(v.dtype)
        for t in range(v.shape[0]):
            if not np.array_equal(np.sort(v[t].ravel()), ranks):
                raise ValueError(f"frame {t} is not a rank permutation")
        v.setflags(write=False)
        object.__setattr__(self, "values", v)

    @property
    def frames(self) -> int:
        return self.values.shape[0]

    @property
    def dims(self) -> tuple[int, int]:
        return self.values.shape[1], self.values.shape[2]


def _rank_values(order_r: np.ndarray, n: int, shape: tuple[int, int]) -> np.ndarray:
    """rank-per-site array -> values (r+0.5)/n reshaped to (H, W) (noise.py:60-62)."""
    return ((order_r.astype(np.float64) + 0.5) / n).reshape(shape).astype(np.float32)


def gen_uniform_noise(h: int, w: int, t: int = 1, seed: int = 0) -> NoiseStack:
    """Independent random rank permutation per frame (noise.py:65-75): the film-sized white-noise
    stack of the compression sweep. Host-side input generation (NumPy's PCG64 stream, as the
    reference), uploaded by the mask kernel like any stack."""
    if h < 8 or w < 8:
        raise ValueError(f"noise dims must be >= 8, got {h}x{w}")
    rng = np.random.default_rng(seed)
    n = h * w
    frames = np.empty((t, h, w), dtype=np.float32)
    for k in range(t):
        frames[k] = _rank_values(rng.permutation(n), n, (h, w))
    return NoiseStack(values=frames, seed=seed)


def save_stack(stack: NoiseStack, path: str | Path) -> None:
    """RNKSTACK cache: magic, (H, W, T, seed, sigma_s, sigma_t), float32 payload."""
    t = stack.values.shape[0]
    h, w = stack.dims
    header = struct.pack(_HEADER, _CACHE_MAGIC, h, w, t, stack.seed, stack.sigma_spatial,
                         stack.sigma_temporal)
    with open(path, "wb") as f:
        f.write(header)
        f.write(np.ascontiguousarray(stack.values, dtype="<f4").tobytes())


def load_stack(path: str | Path) -> NoiseStack:
    blob = Path(path).read_bytes()
    head = struct.calcsize(_HEADER)
    magic, h, w, t, seed, ss, st = struct.unpack(_HEADER, blob[:head])
    if magic != _CACHE_MAGIC:
        raise ValueError(f"not a noise stack cache: {path}")
    values = np.frombuffer(blob[head:], dtype="<f4").reshape(t, h, w).copy()
    return NoiseStack(values=values, seed=seed, sigma_spatial=ss, sigma_temporal=st)


def default_stack(cache_dir: str | Path | None = None, h: int = DEFAULT_TILE,
                  w: int = DEFAULT_TILE, t: int = DEFAULT_FRAMES, seed: int = 1) -> NoiseStack:
    """The pipeline's default STBN tile (noise.py:456-468), read from its RNKSTACK cache."""
    name = f"stbn_{h}x{w}x{t}_s{seed}.noise"
    for d in ([Path(cache_dir)] if cache_dir is not None else []) + [_DATA]:
        if (d / name).exists():
            return load_stack(d / name)
    raise ValueError(
        f"no cached noise stack {name}: generation is an offline step of the reference "
        "(fovray.noise.gen_stbn); cache it with save_stack() and pass cache_dir")


def tile_lookup(stack: NoiseStack, u: int, v: int, frame: int) -> float:
    """Toroidal lookup of one value (noise.py:371-375): a scalar read of the caller's stack (the
    mask kernel performs the same lookup per pixel on the device)."""
    t = stack.values.shape[0]
    h, w = stack.dims
    return float(stack.values[frame % t, v % h, u % w])


def tile_field(stack: NoiseStack, h: int, w: int, frame: int) -> np.ndarray:
    """Frame `frame` of the stack tiled out to an (h, w) field (noise.py:378-384): built on the
    device by fv_tile_field (the mask kernel's lookup), returned as a read-only (h, w) float32 array."""
    import torch

    from . import _lib

    if h < 1 or w < 1:
        raise ValueError(f"dims must be positive, got {(h, w)}")
    ctx = _lib.context()
    ctx.ensure_noise(stack)
    out = torch.empty((h, w), dtype=torch.float32, device="cuda")
    _lib.check(ctx.lib.fv_tile_field(ctx.h, int(frame), int(h), int(w), _lib.ptr(out)))
    a = out.cpu().numpy()
    a.setflags(write=False)
    return a

