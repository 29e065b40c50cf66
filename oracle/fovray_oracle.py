"""CPU ORACLE -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline and
--impl reference legs) may import this module, and only as the checker / the
reported CPU baseline. The product (paper_2209_09965_b200) never calls it.

A restatement of the reference FoVolNet hot path (pkg/src/fovray, NumPy/float64
for masks and marching, float32 for the network) written for checking:

  tau_map / sample_mask / compact          sample_maps.py:62-68, :89-105, :128-132, :161-171
  procedural_volume                        volume.py:112-146 (+ _normalize :75-81)
  camera_basis / render (C, march_oracle.c) volume.py:269-303, renderer.py:88-195
  generate_rays / sample_trilinear / tf_apply volume.py:293-303, :149-180, :201-208
  net_forward (conv/pool/up/K stage)       network.py:183-323, autograd.py:173-359
  psnr / ssim                              metrics.py:40-87

Parity of this restatement with the reference itself is pinned in
tests/test_oracle.py against fixtures produced by running the reference
(tests/golden/make_golden.py), including the reference's own golden SHA-256.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

FULL_BLOCKS = "e64-e64-e80-d96-d80-d64-d64"
DESK_BLOCKS = "e16-e16-e24-d32-d24-d16-d16"
DEFAULT_LUT = np.asarray([
    [0.10, 0.10, 0.35, 0.00], [0.15, 0.35, 0.80, 0.02], [0.10, 0.75, 0.70, 0.12],
    [0.55, 0.85, 0.25, 0.30], [0.95, 0.80, 0.15, 0.55], [0.95, 0.35, 0.10, 0.80],
    [0.90, 0.90, 0.90, 0.95]], dtype=np.float32)


# --------------------------------------------------------------------------- masks
def pixel_scale_for_film(h: int, w: int, fraction: float = 0.45) -> float:
    """sample_maps.py:31-40 with sigma_fast = 0.02."""
    return float(np.sqrt(2.0 / 0.02) / (fraction * min(h, w)))


def tau_map(h, w, focus, sigma, pb, scale) -> np.ndarray:
    """Eq. 1-2 as the reference evaluates them (sample_maps.py:62-68, :101-105), fp64."""
    dx = (np.arange(w, dtype=np.float64) - focus[0])[None, :] * scale
    dy = (np.arange(h, dtype=np.float64) - focus[1])[:, None] * scale
    pf = np.exp(-0.5 * (dx * dx + dy * dy) * sigma)
    return np.minimum(pf + (1.0 - pf) * np.asarray(pb, dtype=np.float64), 1.0)


def noise_field(stack: np.ndarray, h: int, w: int, frame: int) -> np.ndarray:
    """Toroidal lookup stack[frame % T][v % Ht][u % Wt] (noise.py:378-384)."""
    t, th, tw = stack.shape
    return stack[frame % t][(np.arange(h) % th)[:, None], (np.arange(w) % tw)[None, :]]


def sample_mask(stack, h, w, frame, tau) -> np.ndarray:
    """M = float64(N) < tau (sample_maps.py:128-132)."""
    return noise_field(stack, h, w, frame).astype(np.float64) < tau


def compact(bits: np.ndarray) -> np.ndarray:
    """Row-major flat indices v*W+u of the set bits (sample_maps.py:161-171)."""
    return np.flatnonzero(bits.reshape(-1)).astype(np.int64)


def uniform_noise(h: int, w: int, t: int = 1, seed: int = 0) -> np.ndarray:
    """gen_uniform_noise (noise.py:60-75): per frame an independent rank permutation from NumPy's
    PCG64 stream, value (r+0.5)/n as float32 -> (t, h, w)."""
    rng = np.random.default_rng(seed)
    n = h * w
    out = np.empty((t, h, w), np.float32)
    for k in range(t):
        out[k] = ((rng.permutation(n).astype(np.float64) + 0.5) / n).reshape(h, w).astype(np.float32)
    return out


def naive_lanes(bits: np.ndarray, chunk: int = 64) -> np.ndarray:
    """render_sparse_naive's lane set (renderer.py:225-245): flat indices of every pixel of each
    `chunk`-pixel row-major group holding at least one set bit."""
    b = np.asarray(bits, bool).ravel()
    n = b.size
    nc = (n + chunk - 1) // chunk
    pad = np.zeros(nc * chunk, bool)
    pad[:n] = b
    occ = pad.reshape(nc, chunk).any(axis=1)
    return np.flatnonzero(np.repeat(occ, chunk)[:n])


def direct_samples(tau: np.ndarray, count: int, rng: np.random.Generator) -> np.ndarray:
    """draw_direct_samples (sample_maps.py:181-198): inverse-CDF draws over the fp64 tau map ->
    (count, 2) int64 (u, v); duplicates allowed."""
    h, w = tau.shape
    cdf = np.cumsum(tau.ravel())
    cdf /= cdf[-1]
    idx = np.minimum(np.searchsorted(cdf, rng.random(count), side="right"), h * w - 1)
    return np.stack([idx % w, idx // w], axis=1).astype(np.int64)


def load_rnkstack(path) -> np.ndarray:
    import struct

    blob = Path(path).read_bytes()
    head = struct.calcsize("<8sIIIq dd")
    magic, h, w, t, *_ = struct.unpack("<8sIIIq dd", blob[:head])
    assert magic == b"RNKSTACK"
    return np.frombuffer(blob[head:], dtype="<f4").reshape(t, h, w).copy()


# --------------------------------------------------------------------------- volumes
def procedural_volume(kind: str, dims) -> np.ndarray:
    """volume.py:112-146 raw fields at voxel centres, global min-max to float32."""
    nx, ny, nz = dims
    ax = [(np.arange(n) + 0.5) / n * 2.0 - 1.0 for n in (nx, ny, nz)]
    u, v, w = ax[0][None, None, :], ax[1][None, :, None], ax[2][:, None, None]
    r = np.sqrt(u * u + v * v + w * w)
    if kind == "sphere_shells":
        raw = 0.5 * (1.0 + np.cos(2.0 * np.pi * 3.0 * r))
    elif kind == "vortex_field":
        raw = np.sin(3.0 * np.pi * u + 2.0 * v * w) * np.cos(2.0 * np.pi * v - 1.5 * u * w)
        raw = raw + 0.5 * np.cos(4.0 * np.pi * r)
    elif kind == "box_lattice":
        par = (np.floor(2.0 * (u + 1.0)) + np.floor(2.0 * (v + 1.0)) + np.floor(2.0 * (w + 1.0))) % 2.0
        raw = 0.7 * par + 0.3 * (u + 1.0) / 2.0
    else:
        raise ValueError(kind)
    raw = np.ascontiguousarray(np.broadcast_to(raw, (nz, ny, nx)))
    lo, hi = float(raw.min()), float(raw.max())
    data = ((raw - lo) / (hi - lo)).astype(np.float32) if hi > lo else np.zeros(raw.shape, np.float32)
    return data, (lo, hi)


# --------------------------------------------------------------------------- marcher
def build_lib() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "march_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_clib = None


def _lib():
    global _clib
    if _clib is None:
        _clib = C.CDLL(str(build_lib()))
        _clib.oracle_render.restype = None
    return _clib


def camera_basis(position, look_at, up=(0.0, 1.0, 0.0)):
    """Camera.basis (volume.py:269-276), NumPy norms as the reference computes them."""
    fwd = np.subtract(look_at, position, dtype=np.float64)
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    return right, np.cross(right, fwd), fwd


def orbit_camera(i: int, n_frames: int, dims, spacing=(1.0, 1.0, 1.0), radius_factor=2.2,
                 zoom_amplitude=0.35, zoom_periods=2.0, yaw_turns=1.0, pitch_amp_deg=25.0,
                 pitch_periods=1.0):
    """orbit_cameras frame i (renderer.py:317-361) -> (position, look_at)."""
    ext = np.asarray(dims, dtype=np.float64) * np.asarray(spacing, dtype=np.float64)
    center = ext * 0.5
    diag = float(np.linalg.norm(ext))
    s = 0.0 if n_frames <= 1 else i / n_frames
    yaw = 2.0 * np.pi * (yaw_turns * s + 0.0)
    pitch = np.deg2rad(pitch_amp_deg) * np.sin(2.0 * np.pi * pitch_periods * s)
    r = radius_factor * diag * (1.0 + zoom_amplitude * np.sin(2.0 * np.pi * zoom_periods * s))
    pos = center + r * np.array([np.cos(pitch) * np.cos(yaw), np.sin(pitch), np.cos(pitch) * np.sin(yaw)])
    return tuple(pos), tuple(center)


def generate_rays(cam: dict, us, vs):
    """Rays through pixel centres (volume.py:293-303): (origins, unit dirs) (n, 3) fp64."""
    right, up, fwd = camera_basis(cam["position"], cam["look_at"], cam.get("up", (0.0, 1.0, 0.0)))
    tan_half = np.tan(np.deg2rad(cam.get("fov_y", 45.0)) * 0.5)
    aspect = cam["width"] / cam["height"]
    sx = ((np.asarray(us, dtype=np.float64) + 0.5) / cam["width"] * 2.0 - 1.0) * tan_half * aspect
    sy = (1.0 - (np.asarray(vs, dtype=np.float64) + 0.5) / cam["height"] * 2.0) * tan_half
    d = fwd[None, :] + sx[:, None] * right[None, :] + sy[:, None] * up[None, :]
    d = d / np.sqrt((d * d).sum(axis=1, keepdims=True))
    return np.broadcast_to(np.asarray(cam["position"], np.float64), d.shape).copy(), d


def sample_trilinear(data: np.ndarray, spacing, pts) -> np.ndarray:
    """Trilinear value at world points (n, 3), 0 outside [0, ext] (volume.py:149-180); data (nz,ny,nx)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    nz, ny, nx = data.shape
    sp = np.asarray(spacing, dtype=np.float64)
    ext = np.asarray([nx, ny, nz], np.float64) * sp
    inside = np.all((pts >= 0.0) & (pts <= ext), axis=-1)
    q = pts / sp - 0.5
    f = np.floor(q)
    t = q - f
    n = np.asarray([nx, ny, nz])
    i0 = np.clip(f.astype(np.int64), 0, n - 1)
    i1 = np.clip(i0 + 1, 0, n - 1)
    x0, y0, z0 = i0.T
    x1, y1, z1 = i1.T
    tx, ty, tz = t.T
    d = data.astype(np.float64)
    c00 = d[z0, y0, x0] * (1 - tx) + d[z0, y0, x1] * tx
    c10 = d[z0, y1, x0] * (1 - tx) + d[z0, y1, x1] * tx
    c01 = d[z1, y0, x0] * (1 - tx) + d[z1, y0, x1] * tx
    c11 = d[z1, y1, x0] * (1 - tx) + d[z1, y1, x1] * tx
    v = (c00 * (1 - ty) + c10 * ty) * (1 - tz) + (c01 * (1 - ty) + c11 * ty) * tz
    return np.where(inside, v, 0.0)


def tf_apply(lut, s) -> np.ndarray:
    """TransferFunction.apply (volume.py:201-208): clip to [0,1], lerp between LUT rows (fp64)."""
    lut = np.asarray(lut, dtype=np.float32)
    s = np.clip(np.asarray(s, dtype=np.float64), 0.0, 1.0)
    k = lut.shape[0]
    x = s * (k - 1)
    i0 = np.clip(np.floor(x).astype(np.int64), 0, k - 2)
    t = (x - i0)[..., None]
    return lut[i0] * (1 - t) + lut[i0 + 1] * t


def render(volume: np.ndarray, spacing, lut, light, cam: dict, pix=None, step_size=None,
           shadow_step_factor=4.0, early_term_alpha=0.99, background=(0.0, 0.0, 0.0, 0.0),
           ambient=0.25, reference_step=None, shadow_min_transmittance=1e-3, with_counts=False,
           nthreads=None):
    """March pixels `pix` (flat v*W+u; None = all) -> (rgba (n,4) f32, depth (n,) f32[, counts]).

    light: None, ("dir", (x,y,z), intensity) or ("point", (x,y,z), intensity).
    cam: dict(position, look_at, up, fov_y, width, height).
    """
    vol = np.ascontiguousarray(volume, dtype=np.float32)
    nz, ny, nx = vol.shape
    w, h = int(cam["width"]), int(cam["height"])
    base = float(min(spacing))
    step = step_size if step_size is not None else 0.5 * base
    ref = reference_step if reference_step is not None else base
    right, up, fwd = camera_basis(cam["position"], cam["look_at"], cam.get("up", (0.0, 1.0, 0.0)))
    tan_half = np.tan(np.deg2rad(cam.get("fov_y", 45.0)) * 0.5)
    aspect = w / h
    camv = np.concatenate([np.asarray(cam["position"], np.float64), right, up, fwd,
                           [tan_half, aspect]]).astype(np.float64)
    kind, lvec, inten = 0, np.zeros(3), np.ones(3)
    if light is not None:
        if light[0] == "dir":
            kind = 1
            d = -np.asarray(light[1], dtype=np.float64)
            lvec = d / np.linalg.norm(d)
        else:
            kind = 2
            lvec = np.asarray(light[1], dtype=np.float64)
        inten = np.asarray(light[2], dtype=np.float64)
    cfg = np.asarray([step, ref, step * shadow_step_factor, early_term_alpha, ambient,
                      shadow_min_transmittance, *background], dtype=np.float64)
    pix = np.arange(w * h, dtype=np.int64) if pix is None else np.ascontiguousarray(pix, dtype=np.int64)
    n = pix.shape[0]
    rgba = np.zeros((n, 4), dtype=np.float32)
    depth = np.zeros(n, dtype=np.float32)
    counts = np.zeros((n, 2), dtype=np.int64) if with_counts else None
    lut = np.ascontiguousarray(lut, dtype=np.float32)
    dims = np.asarray([nx, ny, nz], dtype=np.int32)
    sp = np.asarray(spacing, dtype=np.float64)

    def P(a):
        return a.ctypes.data_as(C.c_void_p) if a is not None else None

    _lib().oracle_render(P(vol), P(dims), P(sp), P(lut), C.c_int(lut.shape[0]), C.c_int(kind),
                         P(np.ascontiguousarray(lvec, np.float64)), P(np.ascontiguousarray(inten, np.float64)),
                         P(cfg), P(camv), C.c_int(w), C.c_int(h), P(pix), C.c_int64(n), P(rgba),
                         P(depth), P(counts), C.c_int(nthreads or threads()))
    if with_counts:
        return rgba, depth, counts
    return rgba, depth


def render_image(volume, spacing, lut, light, cam: dict, bits=None, **kw):
    """(H,W,4) rgba + (H,W) depth; pixels outside `bits` stay zero (render_sparse_compact)."""
    w, h = int(cam["width"]), int(cam["height"])
    pix = None if bits is None else compact(bits)
    rgba, depth = render(volume, spacing, lut, light, cam, pix=pix, **kw)
    img = np.zeros((h * w, 4), np.float32)
    dep = np.zeros(h * w, np.float32)
    sel = np.arange(h * w) if pix is None else pix
    img[sel] = rgba
    dep[sel] = depth
    return img.reshape(h, w, 4), dep.reshape(h, w)


# --------------------------------------------------------------------------- network (fp32)
def parse_blocks(s: str):
    return [(t[0], int(t[1:])) for t in s.split("-")]


def conv_layout(blocks: str, in_channels: int = 8, recurrent: bool = True):
    """(cin, cout) per D block and K input widths (network.py:128-159)."""
    cfg = parse_blocks(blocks)
    ch = [c for _, c in cfg]
    ne = sum(1 for k, _ in cfg if k == "e")
    nd = len(cfg) - ne
    d_ch = ch[ne:]
    d_in = []
    for j in range(nd):
        inc = ch[ne - 1] if j == 0 else d_ch[j - 1] + ch[ne - j]
        d_in.append(inc + (d_ch[j] if recurrent else 0))
    e_in = [in_channels] + ch[: ne - 1]
    levels = list(range(ne)) + [ne - j for j in range(nd)]
    k_in = [d_ch[ne - lv] for lv in levels]
    return list(zip(e_in, ch[:ne])) + list(zip(d_in, d_ch)), k_in, ne, nd, levels, cfg


def init_params(blocks: str, seed: int, in_channels: int = 8, fp16_weights: bool = False):
    """Seeded He-uniform weights in init_network's draw order (network.py:162-180)."""
    rng = np.random.default_rng(seed)
    layout, k_in, *_ = conv_layout(blocks, in_channels)
    p = {}

    def conv(name, cin, cout, k):
        bound = np.sqrt(6.0 / (cin * k * k))
        w = rng.uniform(-bound, bound, size=(cout, cin, k, k)).astype(np.float32)
        if fp16_weights:
            w = np.clip(w, -65504, 65504).astype(np.float16).astype(np.float32)
        p[name + ".w"] = w
        p[name + ".b"] = np.zeros(cout, np.float32)

    for i, (cin, cout) in enumerate(layout):
        conv(f"D.block{i}.conv1", cin, cout, 3)
        conv(f"D.block{i}.conv2", cout, cout, 3)
    conv("D.head", layout[-1][1], 3, 3)
    for i, cin in enumerate(k_in):
        conv(f"K.block{i}", cin, 9, 1)
    return p


def conv3x3(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Cross-correlation, zero padding 1 (autograd.py:238-276). x (C,H,W) -> (cout,H,W)."""
    return np.ascontiguousarray(conv3x3_hwc(np.ascontiguousarray(np.moveaxis(x, 0, -1)), w, b).transpose(2, 0, 1))


def conv3x3_hwc(x, w: np.ndarray, b: np.ndarray, relu_out: bool = False, band: int = 32) -> np.ndarray:
    """The same conv on a channel-last (H,W,C) image -> (H,W,cout), as nine shifted GEMMs.

    x may be a list of (H,W,C_i) parts: concat_channels (autograd.py:173-185) is done by writing
    the parts into the padded buffer. The zero-padded image is stored with rows of W+2 pixels, so
    tap (ky,kx) of every output pixel in a band of rows is one CONTIGUOUS slice of the flattened
    padded image, offset by ky*(W+2)+kx (the two junk columns per row this computes are dropped).
    No im2col copy is built; the sum over (c, ky, kx) runs in a different order than the
    reference's single sgemm, which moves fp32 results by ~1e-6 (BLAS order is unpinned in the
    reference too). relu_out applies relu (autograd.py:134-141) per band."""
    parts = x if isinstance(x, (list, tuple)) else [x]
    h, wd = parts[0].shape[:2]
    c = sum(p.shape[2] for p in parts)
    wp2 = wd + 2
    cout = w.shape[0]
    xp = np.empty((h + 3, wp2, c), np.float32)
    xp[0] = 0.0
    xp[h + 1:] = 0.0
    xp[:, 0] = 0.0
    xp[:, wd + 1] = 0.0
    c0 = 0
    for p in parts:
        xp[1:h + 1, 1:wd + 1, c0:c0 + p.shape[2]] = p
        c0 += p.shape[2]
    flat = xp.reshape(-1, c)
    taps = [np.ascontiguousarray(w[:, :, t // 3, t % 3].T, dtype=np.float32) for t in range(9)]
    bias = b.astype(np.float32)
    out = np.empty((h, wd, cout), np.float32)
    tmp = None
    for r0 in range(0, h, band):
        rows = min(band, h - r0)
        n = rows * wp2
        acc = flat[r0 * wp2:r0 * wp2 + n] @ taps[0]
        if tmp is None or tmp.shape[0] != n:
            tmp = np.empty((n, cout), np.float32)
        for t in range(1, 9):
            o = (r0 + t // 3) * wp2 + t % 3
            np.matmul(flat[o:o + n], taps[t], out=tmp)
            acc += tmp
        acc += bias
        if relu_out:
            np.maximum(acc, 0.0, out=acc)
        out[r0:r0 + rows] = acc.reshape(rows, wp2, cout)[:, :wd]
    return out


def relu(x):
    return x * (x > 0)


def pool2(x):
    """avg_pool2 (autograd.py:279-291) on (C,H,W)."""
    return 0.25 * (x[:, 0::2, 0::2] + x[:, 1::2, 0::2] + x[:, 0::2, 1::2] + x[:, 1::2, 1::2])


def pool2_hwc(x):
    return 0.25 * (x[0::2, 0::2] + x[1::2, 0::2] + x[0::2, 1::2] + x[1::2, 1::2])


def _up2_axis(d, ax):
    """Half-pixel bilinear x2 along one axis, edge clamp (autograd.py:294-305):
    out[2i] = 0.25*d[i-1] + 0.75*d[i], out[2i+1] = 0.75*d[i] + 0.25*d[i+1] (clamped)."""
    d = np.moveaxis(d, ax, 0)
    n = d.shape[0]
    out = np.empty((2 * n,) + d.shape[1:], dtype=d.dtype)
    q = 0.75 * d
    ev, od = out[0::2], out[1::2]
    np.multiply(d[:1], 0.25, out=ev[:1])
    np.multiply(d[:-1], 0.25, out=ev[1:])
    ev += q
    np.multiply(d[1:], 0.25, out=od[:-1])
    np.multiply(d[-1:], 0.25, out=od[-1:])
    od += q  # (0.75*d + 0.25*nxt: the same two rounded products and one rounded sum)
    return np.moveaxis(out, 0, ax)


def up2(x):
    """upsample_bilinear2 (autograd.py:322-329) on (C,H,W): rows then columns."""
    return _up2_axis(_up2_axis(x, 1), 2)


def up2_hwc(x):
    return _up2_axis(_up2_axis(x, 0), 1)


def kernel_filter(img, logits):
    """softmax over 9 taps then per-pixel 3x3 filter, zero padding (autograd.py:188-199, :332-359).
    img (3,H,W), logits (9,H,W)."""
    return kernel_filter_hwc(np.moveaxis(img, 0, -1), np.moveaxis(logits, 0, -1)).transpose(2, 0, 1)


def kernel_filter_hwc(img, logits):
    m = logits.max(axis=-1, keepdims=True)
    e = np.exp(logits - m)
    k = e / e.sum(axis=-1, keepdims=True)
    h, w = img.shape[:2]
    ip = np.pad(img, ((1, 1), (1, 1), (0, 0)))
    out = np.zeros_like(img)
    for j in range(9):
        dy, dx = divmod(j, 3)
        out += k[..., j:j + 1] * ip[dy:dy + h, dx:dx + w]
    return out


def net_forward(params: dict, blocks: str, x: np.ndarray, state: dict | None, use_k: bool = True):
    """forward_full for one frame (network.py:296-323). x (C,H,W) float32 rgba[+mask].

    state: None or {"hidden": [arrays (C,Hp/s,Wp/s)], "prev": (3,Hp,Wp)}.
    returns (O (3,H,W), O_d (3,H,W), new_state); the state's arrays are (C,h,w) views of
    channel-last buffers (the whole forward runs channel-last, see conv3x3_hwc).
    """
    layout, k_in, ne, nd, levels, cfg = conv_layout(blocks)
    c, h, w = x.shape
    div = 2 ** ne
    hp, wp = -(-h // div) * div, -(-w // div) * div
    cur = np.zeros((hp, wp, c + 3), np.float32)
    cur[:h, :w, :c] = np.moveaxis(x, 0, -1)
    if state is not None:
        cur[..., c:] = np.moveaxis(state["prev"], 0, -1)
    P = params

    def block(t, i):
        t = conv3x3_hwc(t, P[f"D.block{i}.conv1.w"], P[f"D.block{i}.conv1.b"], relu_out=True)
        return conv3x3_hwc(t, P[f"D.block{i}.conv2.w"], P[f"D.block{i}.conv2.b"], relu_out=True)

    skips = []
    for i in range(ne):
        cur = block(cur, i)
        skips.append(cur)
        cur = pool2_hwc(cur)
    hd = []
    for j in range(nd):
        parts = [up2_hwc(cur), skips[ne - j]] if j > 0 else [cur]
        parts.append(np.zeros(parts[0].shape[:2] + (layout[ne + j][1],), np.float32) if state is None
                     else np.moveaxis(state["hidden"][j], 0, -1))
        cur = block(parts, ne + j)
        hd.append(cur)
    od = conv3x3_hwc(hd[-1], P["D.head.w"], P["D.head.b"])
    img = od
    if use_k:
        by_level = {ne - j: hd[j] for j in range(nd)}
        for i, lv in enumerate(levels):
            hdl = by_level[lv]
            logits = hdl @ np.ascontiguousarray(P[f"K.block{i}.w"][:, :, 0, 0].T) + P[f"K.block{i}.b"]
            img = kernel_filter_hwc(img, logits)
            if cfg[i][0] == "e":
                img = pool2_hwc(img)
            elif i < len(cfg) - 1:
                img = up2_hwc(img)
    chw = lambda a: a.transpose(2, 0, 1)  # noqa: E731
    return (np.ascontiguousarray(chw(img[:h, :w])), np.ascontiguousarray(chw(od[:h, :w])),
            {"hidden": [chw(t) for t in hd], "prev": chw(od)})


# --------------------------------------------------------------------------- metrics
def psnr(a, b, peak=1.0) -> float:
    """metrics.psnr (metrics.py:40-49): joint RGB, 100 dB cap."""
    a = np.asarray(a, np.float64)[..., :3]
    b = np.asarray(b, np.float64)[..., :3]
    mse = float(np.mean((a - b) ** 2))
    if mse == 0.0:
        return 100.0
    return min(10.0 * float(np.log10(peak * peak / mse)), 100.0)


def ssim(a, b) -> float:
    """metrics.ssim (metrics.py:74-87): Rec.601 luma, 11x11 Gaussian (sigma 1.5), valid windows."""
    from numpy.lib.stride_tricks import sliding_window_view

    def luma(img):
        img = np.asarray(img, np.float64)
        return 0.299 * img[..., 0] + 0.587 * img[..., 1] + 0.114 * img[..., 2]

    d = np.arange(11, dtype=np.float64) - 5.0
    k = np.exp(-(d * d) / (2 * 1.5 * 1.5))
    k /= k.sum()

    def filt(im):
        rows = sliding_window_view(im, 11, axis=0) @ k
        return sliding_window_view(rows, 11, axis=1) @ k

    la, lb = luma(a), luma(b)
    mu_a, mu_b = filt(la), filt(lb)
    va = filt(la * la) - mu_a * mu_a
    vb = filt(lb * lb) - mu_b * mu_b
    cov = filt(la * lb) - mu_a * mu_b
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    s = ((2 * mu_a * mu_b + c1) * (2 * cov + c2)) / ((mu_a * mu_a + mu_b * mu_b + c1) * (va + vb + c2))
    return float(s.mean())


def _ssim_maps(la, lb):
    from numpy.lib.stride_tricks import sliding_window_view

    d = np.arange(11, dtype=np.float64) - 5.0
    k = np.exp(-(d * d) / (2 * 1.5 * 1.5))
    k /= k.sum()

    def filt(im):
        rows = sliding_window_view(im, 11, axis=0) @ k
        return sliding_window_view(rows, 11, axis=1) @ k

    mu_a, mu_b = filt(la), filt(lb)
    va = filt(la * la) - mu_a * mu_a
    vb = filt(lb * lb) - mu_b * mu_b
    cov = filt(la * lb) - mu_a * mu_b
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    cs = (2 * cov + c2) / (va + vb + c2)
    lum = (2 * mu_a * mu_b + c1) / (mu_a * mu_a + mu_b * mu_b + c1)
    return lum, cs


def _luma(img):
    img = np.asarray(img, np.float64)
    if img.ndim == 2:
        return img
    return 0.299 * img[..., 0] + 0.587 * img[..., 1] + 0.114 * img[..., 2]


def msssim(a, b) -> float:
    """metrics.msssim (metrics.py:96-130): scales while the coarse image keeps an 11px window,
    weights renormalised, contrast-structure means clamped at 0, 2x2 mean downsampling."""
    wts_all = (0.0448, 0.2856, 0.3001, 0.2363, 0.1333)
    la, lb = _luma(a), _luma(b)
    m, size = 1, min(la.shape)
    while m < len(wts_all) and size // 2 >= 11:
        size //= 2
        m += 1
    wts = np.asarray(wts_all[:m])
    wts = wts / wts.sum()
    value = 1.0
    for j in range(m):
        lum, cs = _ssim_maps(la, lb)
        stat = float((lum * cs).mean()) if j == m - 1 else float(cs.mean())
        value *= max(stat, 0.0) ** wts[j]
        if j < m - 1:
            h, w = la.shape
            la = la[: h // 2 * 2, : w // 2 * 2]
            lb = lb[: h // 2 * 2, : w // 2 * 2]
            la = 0.25 * (la[0::2, 0::2] + la[1::2, 0::2] + la[0::2, 1::2] + la[1::2, 1::2])
            lb = 0.25 * (lb[0::2, 0::2] + lb[1::2, 0::2] + lb[0::2, 1::2] + lb[1::2, 1::2])
    return float(value)


def tpsnr(seq_a, seq_b) -> np.ndarray:
    """metrics.tpsnr (metrics.py:133-148): PSNR of (d+1)/2 temporal differences."""
    out = np.empty(len(seq_a) - 1)
    for i in range(1, len(seq_a)):
        da = (np.asarray(seq_a[i], np.float64)[..., :3] - np.asarray(seq_a[i - 1], np.float64)[..., :3] + 1.0) / 2.0
        db = (np.asarray(seq_b[i], np.float64)[..., :3] - np.asarray(seq_b[i - 1], np.float64)[..., :3] + 1.0) / 2.0
        out[i - 1] = psnr(da, db)
    return out


def threads() -> int:
    return len(os.sched_getaffinity(0))
