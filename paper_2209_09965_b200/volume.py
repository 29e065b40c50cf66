"""Volume data, transfer functions, cameras and lights (device-resident volumes).

Drop-in for pkg/src/fovray/volume.py. A VolumeGrid's scalar field lives on the GPU
as a (nz, ny, nx) float32 tensor in [0,1] (the reference layout, volume.py:47-72);
make_procedural_volume (volume.py:112-146) generates it with a CUDA kernel in fp64
and load_raw_volume (volume.py:84-109) normalises raw files on the device.
Cameras, lights and transfer functions are small host value types.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib

_DTYPES = {"uint8": np.uint8, "float32": np.dtype("<f4")}
_KINDS = {"sphere_shells": 0, "vortex_field": 1, "box_lattice": 2}


@dataclass(frozen=True)
class VolumeMeta:
    """Sidecar descriptor for a raw volume file (volume.py:24-44)."""

    dims: tuple[int, int, int]
    dtype: str = "uint8"
    spacing: tuple[float, float, float] = (1.0, 1.0, 1.0)

    @staticmethod
    def from_file(path: str | Path) -> "VolumeMeta":
        spec = json.loads(Path(path).read_text())
        return VolumeMeta(dims=tuple(int(d) for d in spec["dims"]), dtype=spec.get("dtype", "uint8"),
                          spacing=tuple(float(s) for s in spec.get("spacing", (1.0, 1.0, 1.0))))

    def to_file(self, path: str | Path) -> None:
        Path(path).write_text(json.dumps({"dims": list(self.dims), "dtype": self.dtype,
                                          "spacing": list(self.spacing)}))


class VolumeGrid:
    """Scalar field on a regular grid, values in [0,1], stored on the GPU."""

    def __init__(self, dims, spacing, data, value_range, *, _validated: bool = False):
        import torch

        nx, ny, nz = (int(d) for d in dims)
        if min(nx, ny, nz) < 2:
            raise ValueError(f"volume dims must all be >= 2, got {tuple(dims)}")
        self.dims = (nx, ny, nz)
        self.spacing = tuple(float(s) for s in spacing)
        t = data if isinstance(data, torch.Tensor) else torch.as_tensor(np.asarray(data, dtype=np.float32))
        t = t.to(device="cuda", dtype=torch.float32).contiguous()
        if tuple(t.shape) != (nz, ny, nx):
            raise ValueError(f"data shape {tuple(t.shape)} does not match dims {self.dims}")
        if not _validated and t.numel() and (float(t.min()) < 0.0 or float(t.max()) > 1.0):
            raise ValueError("volume data must be normalized to [0,1]")
        self._data = t
        self.value_range = tuple(float(v) for v in value_range)
        self._handles = {}

    @property
    def data_dev(self):
        """(nz, ny, nx) float32 CUDA tensor."""
        return self._data

    @property
    def data(self) -> np.ndarray:
        a = self._data.cpu().numpy()
        a.setflags(write=False)
        return a

    @property
    def extent(self) -> np.ndarray:
        return np.asarray(self.dims, dtype=np.float64) * np.asarray(self.spacing, dtype=np.float64)

    def center(self) -> np.ndarray:
        return self.extent * 0.5

    def handle(self, ctx: _lib.Context, tf: "TransferFunction"):
        """fv_volume bound to this grid's memory and `tf` (uploaded once per device).

        The handle (and the marcher's quad texture it builds on first use, 4 floats per voxel:
        2 GiB at 512^3) is shared by every context on the device -- the texture build synchronises
        the stream it runs on, so later contexts' streams only ever read it."""
        key = (int(ctx.device), id(tf))
        h = self._handles.get(key)
        if h is None:
            h = C.c_void_p()
            sp = (C.c_double * 3)(*self.spacing)
            _lib.check(ctx.lib.fv_volume_wrap(ctx.h, *self.dims, sp, _lib.ptr(self._data), C.byref(h)))
            lut = np.ascontiguousarray(tf.lut, dtype=np.float32)
            _lib.check(ctx.lib.fv_volume_set_tf(ctx.h, h, lut.ctypes.data_as(C.c_void_p), lut.shape[0]))
            self._handles[key] = (h, ctx, tf)
        return self._handles[key][0]

    def __del__(self):
        for h, ctx, _ in getattr(self, "_handles", {}).values():
            try:
                ctx.lib.fv_volume_destroy(h)
            except Exception:
                pass


def load_raw_volume(path: str | Path, meta: VolumeMeta) -> VolumeGrid:
    """Load a little-endian raw volume and min-max normalise it (volume.py:84-109)."""
    import torch

    if meta.dtype not in _DTYPES:
        raise ValueError(f"unsupported dtype {meta.dtype!r}; expected one of {sorted(_DTYPES)}")
    nx, ny, nz = meta.dims
    elem = np.dtype(_DTYPES[meta.dtype])
    expected = nx * ny * nz * elem.itemsize
    blob = Path(path).read_bytes()
    if len(blob) != expected:
        raise ValueError(f"size mismatch for {path}: expected {expected} bytes "
                         f"({nx}x{ny}x{nz} {meta.dtype}), got {len(blob)}")
    raw = torch.as_tensor(np.frombuffer(blob, dtype=elem).copy(), device="cuda")
    # NaN scan, global min/max and the fp64 normalisation run in libfovnet (fv_volume_from_raw)
    ctx = _lib.context()
    out = torch.empty((nz, ny, nx), dtype=torch.float32, device="cuda")
    h = C.c_void_p()
    sp = (C.c_double * 3)(*meta.spacing)
    _lib.check(ctx.lib.fv_volume_wrap(ctx.h, nx, ny, nz, sp, _lib.ptr(out), C.byref(h)))
    try:
        vr = (C.c_double * 2)()
        nan_at = C.c_int64()
        _lib.check(ctx.lib.fv_volume_from_raw(ctx.h, h, _lib.ptr(raw), 0 if meta.dtype == "uint8" else 1, vr,
                                              C.byref(nan_at)))
    finally:
        ctx.lib.fv_volume_destroy(h)
    return VolumeGrid(meta.dims, meta.spacing, out, (vr[0], vr[1]), _validated=True)


def make_procedural_volume(kind: str, dims: tuple[int, int, int],
                           spacing: tuple[float, float, float] = (1.0, 1.0, 1.0)) -> VolumeGrid:
    """Deterministic test volume generated on the GPU (volume.py:112-146)."""
    import torch

    if min(dims) < 8:
        raise ValueError(f"procedural dims must be >= 8 per axis, got {dims}")
    if kind not in _KINDS:
        raise ValueError(f"unknown procedural volume kind {kind!r}")
    ctx = _lib.context()
    nx, ny, nz = dims
    out = torch.empty((nz, ny, nx), dtype=torch.float32, device="cuda")
    h = C.c_void_p()
    sp = (C.c_double * 3)(*spacing)
    _lib.check(ctx.lib.fv_volume_wrap(ctx.h, nx, ny, nz, sp, _lib.ptr(out), C.byref(h)))
    try:
        vr = (C.c_double * 2)()
        _lib.check(ctx.lib.fv_volume_procedural(ctx.h, h, _KINDS[kind], vr))
    finally:
        ctx.lib.fv_volume_destroy(h)
    return VolumeGrid(dims, spacing, out, (vr[0], vr[1]), _validated=True)


@dataclass(frozen=True)
class TransferFunction:
    """RGBA lookup table over [0,1], K >= 2 entries (volume.py:184-242)."""

    lut: np.ndarray

    def __post_init__(self):
        lut = np.asarray(self.lut, dtype=np.float32)
        if lut.ndim != 2 or lut.shape[1] != 4 or lut.shape[0] < 2:
            raise ValueError(f"transfer function lut must be (K>=2, 4), got {lut.shape}")
        if lut.min() < 0.0 or lut.max() > 1.0:
            raise ValueError("transfer function entries must lie in [0,1]")
        if lut.shape[0] > 256:
            raise ValueError("transfer function lut is limited to 256 entries on the device")
        lut = lut.copy()
        lut.setflags(write=False)
        object.__setattr__(self, "lut", lut)

    def __hash__(self):
        return id(self)

    def apply(self, s) -> np.ndarray:
        """Map scalars s (any shape) to RGBA, shape s.shape + (4,) (volume.py:201-208): clip to [0,1],
        linear interpolation between LUT entries, fp64 on the device (fv_tf_apply)."""
        import torch

        a = np.asarray(s, dtype=np.float64)
        st = torch.as_tensor(np.ascontiguousarray(a).reshape(-1), device="cuda")
        lut = torch.as_tensor(np.ascontiguousarray(self.lut), device="cuda")
        out = torch.empty((st.numel(), 4), dtype=torch.float64, device="cuda")
        ctx = _lib.context()
        _lib.check(ctx.lib.fv_tf_apply(ctx.h, _lib.ptr(lut), int(self.lut.shape[0]), _lib.ptr(st), int(st.numel()),
                                       _lib.ptr(out)))
        return out.cpu().numpy().reshape(a.shape + (4,))

    @staticmethod
    def from_file(path: str | Path) -> "TransferFunction":
        rows = []
        for line in Path(path).read_text().splitlines():
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            vals = [float(tok) for tok in line.split()]
            if len(vals) != 4:
                raise ValueError(f"transfer function line needs 4 floats, got {line!r}")
            rows.append(vals)
        return TransferFunction(lut=np.asarray(rows, dtype=np.float32))

    def to_file(self, path: str | Path) -> None:
        Path(path).write_text("\n".join(" ".join(f"{c:.6f}" for c in row) for row in self.lut) + "\n")

    @staticmethod
    def default() -> "TransferFunction":
        # cool-to-warm ramp, alpha rising with density (volume.py:227-242)
        return TransferFunction(lut=np.asarray([
            [0.10, 0.10, 0.35, 0.00],
            [0.15, 0.35, 0.80, 0.02],
            [0.10, 0.75, 0.70, 0.12],
            [0.55, 0.85, 0.25, 0.30],
            [0.95, 0.80, 0.15, 0.55],
            [0.95, 0.35, 0.10, 0.80],
            [0.90, 0.90, 0.90, 0.95],
        ], dtype=np.float32))


@dataclass(frozen=True)
class Camera:
    """Pinhole camera through pixel centres (volume.py:245-276)."""

    position: tuple[float, float, float]
    look_at: tuple[float, float, float]
    up: tuple[float, float, float] = (0.0, 1.0, 0.0)
    fov_y: float = 45.0
    width: int = 320
    height: int = 180

    def __post_init__(self):
        if not (0.0 < self.fov_y < 180.0):
            raise ValueError(f"fov_y must be in (0, 180) degrees, got {self.fov_y}")
        if self.width < 1 or self.height < 1:
            raise ValueError("film dims must be positive")
        fwd = np.subtract(self.look_at, self.position, dtype=np.float64)
        n = np.linalg.norm(fwd)
        if n == 0.0:
            raise ValueError("camera position and look_at coincide")
        if np.linalg.norm(np.cross(fwd / n, np.asarray(self.up, dtype=np.float64))) < 1e-9:
            raise ValueError("up vector is parallel to the view direction")

    def basis(self):
        fwd = np.subtract(self.look_at, self.position, dtype=np.float64)
        fwd /= np.linalg.norm(fwd)
        right = np.cross(fwd, np.asarray(self.up, dtype=np.float64))
        right /= np.linalg.norm(right)
        return right, np.cross(right, fwd), fwd

    def c_struct(self) -> _lib.FvCamera:
        c = _lib.FvCamera()
        for i in range(3):
            c.position[i] = float(self.position[i])
            c.look_at[i] = float(self.look_at[i])
            c.up[i] = float(self.up[i])
        c.fov_y = float(self.fov_y)
        c.width, c.height = int(self.width), int(self.height)
        return c


@dataclass(frozen=True)
class Light:
    """Directional or point light (volume.py:306-328)."""

    direction: tuple[float, float, float] | None = None
    position: tuple[float, float, float] | None = None
    intensity: tuple[float, float, float] = (1.0, 1.0, 1.0)

    def __post_init__(self):
        if (self.direction is None) == (self.position is None):
            raise ValueError("light needs exactly one of direction or position")
        vec = self.direction if self.direction is not None else self.position
        if not np.all(np.isfinite(vec)):
            raise ValueError("light vector must be finite")
        if not np.all(np.isfinite(self.intensity)) or min(self.intensity) < 0:
            raise ValueError("light intensity must be finite and >= 0")
        if self.direction is not None and np.linalg.norm(self.direction) == 0:
            raise ValueError("light direction must be nonzero")

    def c_struct(self) -> _lib.FvLight:
        l = _lib.FvLight()
        if self.direction is not None:
            l.kind = _lib.LIGHT_DIRECTIONAL
            vec = self.direction
        else:
            l.kind = _lib.LIGHT_POINT
            vec = self.position
        for i in range(3):
            l.vec[i] = float(vec[i])
            l.intensity[i] = float(self.intensity[i])
        return l


_SAMPLING_TF = None


def _sampling_tf() -> TransferFunction:
    global _SAMPLING_TF
    if _SAMPLING_TF is None:
        _SAMPLING_TF = TransferFunction.default()
    return _SAMPLING_TF


def generate_rays(cam: Camera, us, vs) -> tuple[np.ndarray, np.ndarray]:
    """Rays through pixel centres (volume.py:293-303): (origins, unit directions), shape (n, 3) fp64,
    computed by fv_generate_rays (the marcher's in-kernel ray generation)."""
    import torch

    u = np.asarray(us).reshape(-1)
    v = np.asarray(vs).reshape(-1)
    if u.shape != v.shape:
        raise ValueError("us and vs must have the same length")
    n = int(u.size)
    tu = torch.as_tensor(u.astype(np.int32), device="cuda")
    tv = torch.as_tensor(v.astype(np.int32), device="cuda")
    o = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    d = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    camc = cam.c_struct()
    _lib.check(ctx.lib.fv_generate_rays(ctx.h, C.byref(camc), _lib.ptr(tu), _lib.ptr(tv), n, _lib.ptr(o),
                                        _lib.ptr(d)))
    return o.cpu().numpy(), d.cpu().numpy()


def sample_trilinear(vol: VolumeGrid, p) -> np.ndarray:
    """Trilinearly interpolated value at world point(s) p, 0 outside the box (volume.py:149-180);
    fp64 on the device (fv_sample_trilinear). p has shape (..., 3); the result has shape (...)."""
    import torch

    pts = np.asarray(p, dtype=np.float64)
    scalar = pts.ndim == 1
    flat = np.ascontiguousarray(np.atleast_2d(pts).reshape(-1, 3))
    tp = torch.as_tensor(flat, device="cuda")
    out = torch.empty((flat.shape[0],), dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    h = vol.handle(ctx, _sampling_tf())  # (any TF: the handle is only the grid's view here)
    _lib.check(ctx.lib.fv_sample_trilinear(ctx.h, h, _lib.ptr(tp), int(flat.shape[0]), _lib.ptr(out)))
    res = out.cpu().numpy().reshape(np.atleast_2d(pts).shape[:-1])
    return res[0] if scalar else res

