"""Hybrid reconstruction network (W-Net inference) on the GPU.

Drop-in for the inference surface of pkg/src/fovray/network.py: NetConfig
(:37-91), init_network (:162-180, identical seeded weights), load_network /
save_network (FVRCKPT1, :333-357 and autograd.py:530-567), reset_state (:118-119)
and forward_full (:296-323). The forward runs in libfovnet: every 3x3 conv is a
tcgen05 implicit GEMM over fp16 NC8HW8 activations with fp32 accumulation,
encoder pooling and the channel concats are fused into the convs, and the
recurrent state stays on the device between frames. Weights are stored as
binary16 (the reference's fp16 storage emulation, bench._quantized_net).
"""
from __future__ import annotations

import ctypes as C
import json
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib

DESK_BLOCKS = "e16-e16-e24-d32-d24-d16-d16"
FULL_BLOCKS = "e64-e64-e80-d96-d80-d64-d64"


@dataclass(frozen=True)
class NetConfig:
    block_config: tuple[tuple[str, int], ...]
    kernel_size: int = 3
    predicted_kernel: int = 3
    recurrent: bool = True
    include_mask_channel: bool = True

    @staticmethod
    def from_string(blocks: str = DESK_BLOCKS, **kwargs) -> "NetConfig":
        parsed = []
        for tok in blocks.split("-"):
            kind, ch = tok[0], int(tok[1:])
            if kind not in ("e", "d") or ch <= 0:
                raise ValueError(f"bad block token {tok!r}")
            parsed.append((kind, ch))
        return NetConfig(block_config=tuple(parsed), **kwargs)

    def __post_init__(self):
        kinds = [k for k, _ in self.block_config]
        n_e, n_d = kinds.count("e"), kinds.count("d")
        if kinds != ["e"] * n_e + ["d"] * n_d:
            raise ValueError("block config must list e-blocks then d-blocks")
        if n_e != n_d - 1:
            raise ValueError(
                f"structural encoder count (e-blocks + bottleneck = {n_e + 1}) must be one "
                f"more than decoder count ({n_d - 1}); got {n_e} e and {n_d} d blocks")
        if self.predicted_kernel % 2 == 0 or self.kernel_size % 2 == 0:
            raise ValueError("kernel sizes must be odd")

    @property
    def n_enc(self) -> int:
        return sum(1 for k, _ in self.block_config if k == "e")

    @property
    def n_dec(self) -> int:
        return len(self.block_config) - self.n_enc

    @property
    def divisor(self) -> int:
        return 2 ** self.n_enc

    @property
    def in_channels(self) -> int:
        return 4 + (1 if self.include_mask_channel else 0) + (3 if self.recurrent else 0)

    def channels(self) -> list[int]:
        return [c for _, c in self.block_config]

    def to_string(self) -> str:
        return "-".join(f"{k}{c}" for k, c in self.block_config)


def _conv_channels(config: NetConfig):
    """Per-D-block (in, out) widths and K's input widths (network.py:128-149)."""
    ch = config.channels()
    n_e = config.n_enc
    d_ch = ch[n_e:]
    d_in = []
    for j in range(config.n_dec):
        inc = ch[n_e - 1] if j == 0 else d_ch[j - 1] + ch[n_e - j]
        if config.recurrent:
            inc += d_ch[j]
        d_in.append(inc)
    e_in = [config.in_channels] + ch[: n_e - 1]
    levels = _block_levels(config)
    hd = {config.n_enc - j: d_ch[j] for j in range(config.n_dec)}
    return list(zip(e_in, ch[:n_e])) + list(zip(d_in, d_ch)), [hd[lv] for lv in levels]


def _block_levels(config: NetConfig) -> list[int]:
    return list(range(config.n_enc)) + [config.n_enc - j for j in range(config.n_dec)]


def _he_uniform(rng: np.random.Generator, shape) -> np.ndarray:
    fan_in = int(np.prod(shape[1:]))
    bound = np.sqrt(6.0 / fan_in)
    return rng.uniform(-bound, bound, size=shape).astype(np.float32)


class DeviceTensor:
    """Result tensor resident on the GPU; `.data` copies to NumPy on first access."""

    def __init__(self, dev):
        self.dev = dev
        self._host = None

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = self.dev.cpu().numpy()
        return self._host

    @property
    def shape(self):
        return tuple(self.dev.shape) if self.dev is not None else tuple(self._host.shape)


def _arr(v) -> np.ndarray:
    return np.asarray(getattr(v, "data", v), dtype=np.float32)


class WNetParams:
    """Network config + named float32 parameters (host), uploaded per device context."""

    def __init__(self, config: NetConfig, params: dict):
        self.config = config
        self.params = params
        self._dev = {}

    def named_arrays(self) -> dict[str, np.ndarray]:
        return {name: _arr(p) for name, p in self.params.items()}

    def handle(self, ctx: _lib.Context):
        """fv_net for this context; re-uploaded when any parameter object changed."""
        fp = tuple((n, id(p)) for n, p in self.params.items())
        ent = self._dev.get(id(ctx))
        if ent is not None and ent[1] == fp:
            return ent[0]
        if ent is not None:
            ctx.lib.fv_net_destroy(ent[0])
        h = C.c_void_p()
        cfg = self.config
        _lib.check(ctx.lib.fv_net_create(ctx.h, cfg.to_string().encode(), cfg.predicted_kernel,
                                         int(cfg.recurrent), int(cfg.include_mask_channel), C.byref(h)))
        for name, p in self.params.items():
            a = np.ascontiguousarray(_arr(p))
            _lib.check(ctx.lib.fv_net_set_param(ctx.h, h, name.encode(), a.ctypes.data_as(C.c_void_p),
                                                a.size))
        self._dev[id(ctx)] = (h, fp, ctx)
        return h

    def __del__(self):
        for h, _, ctx in getattr(self, "_dev", {}).values():
            try:
                ctx.lib.fv_net_destroy(h)
            except Exception:
                pass


def init_network(config: NetConfig, seed: int = 0) -> WNetParams:
    """He-uniform conv weights, zero biases; same values as network.init_network (:162-180)."""
    rng = np.random.default_rng(seed)
    k = config.kernel_size
    params: dict[str, np.ndarray] = {}

    def conv(name, cin, cout, ksz):
        params[f"{name}.w"] = _he_uniform(rng, (cout, cin, ksz, ksz))
        params[f"{name}.b"] = np.zeros(cout, dtype=np.float32)

    d_blocks, k_in = _conv_channels(config)
    for i, (cin, cout) in enumerate(d_blocks):
        conv(f"D.block{i}.conv1", cin, cout, k)
        conv(f"D.block{i}.conv2", cout, cout, k)
    conv("D.head", d_blocks[-1][1], 3, k)
    kf = config.predicted_kernel
    for i, cin in enumerate(k_in):
        conv(f"K.block{i}", cin, kf * kf, 1)
    return WNetParams(config=config, params=params)


class _DevState:
    def __init__(self, ctx, net_handle, h, w):
        self.ctx = ctx
        self.net_handle = net_handle
        hd = C.c_void_p()
        _lib.check(ctx.lib.fv_state_create(ctx.h, net_handle, h, w, C.byref(hd)))
        self.h = hd
        dims = [C.c_int() for _ in range(4)]
        _lib.check(ctx.lib.fv_state_dims(hd, *[C.byref(d) for d in dims]))
        self.H, self.W, self.Hp, self.Wp = (d.value for d in dims)

    def read(self, which: int) -> np.ndarray:
        n = C.c_int64()
        _lib.check(self.ctx.lib.fv_state_read(self.ctx.h, self.h, which, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        _lib.check(self.ctx.lib.fv_state_read(self.ctx.h, self.h, which, out.ctypes.data_as(C.c_void_p),
                                              n.value, C.byref(n)))
        return out

    def __del__(self):
        try:
            self.ctx.lib.fv_state_destroy(self.h)
        except Exception:
            pass


class RecurrentState:
    """Hidden tensors of D's decoder blocks plus O_d feedback (network.py:103-115).

    The device copy advances in place; forward_full hands back a new RecurrentState
    sharing it and retires the one it consumed.
    """

    def __init__(self, film_dims, hidden=None, prev_output=None, *, _dev=None, _config=None):
        self.film_dims = tuple(film_dims)
        self._init_hidden = hidden
        self._init_prev = prev_output
        self._dev = _dev
        self._config = _config
        self._consumed = False

    @property
    def hidden(self):
        if self._dev is None:
            return self._init_hidden
        cfg = self._config
        out = []
        d_ch = cfg.channels()[cfg.n_enc:]
        for j in range(cfg.n_dec):
            s = 2 ** (cfg.n_enc - j)
            a = self._dev.read(j).reshape(1, d_ch[j], self._dev.Hp // s, self._dev.Wp // s)
            out.append(DeviceTensor.__new__(DeviceTensor))
            out[-1].dev, out[-1]._host = None, a
        return out

    @property
    def prev_output(self):
        if self._dev is None:
            return self._init_prev
        t = DeviceTensor.__new__(DeviceTensor)
        t.dev, t._host = None, self._dev.read(-1).reshape(1, 3, self._dev.Hp, self._dev.Wp)
        return t


def reset_state(config: NetConfig, dims: tuple[int, int]) -> RecurrentState:
    return RecurrentState(film_dims=tuple(dims), hidden=[None] * config.n_dec, prev_output=None,
                          _config=config)


def _bind_state(net: WNetParams, state: RecurrentState, ctx, handle) -> _DevState:
    if state._consumed:
        raise ValueError("this recurrent state was consumed by a later forward; carry the returned state")
    h, w = state.film_dims
    if state._dev is not None and state._dev.net_handle.value == handle.value and state._dev.ctx is ctx:
        return state._dev
    dev = _DevState(ctx, handle, h, w)
    # explicit initial tensors (reference RecurrentState built by hand)
    hidden = state.hidden if state._dev is None else state.hidden
    if hidden is not None:
        for j, t in enumerate(hidden):
            if t is None:
                continue
            a = np.ascontiguousarray(_arr(t))
            if a.shape[0] != 1:
                raise ValueError(f"recurrent state batch {a.shape[0]} incompatible with input batch 1")
            _lib.check(ctx.lib.fv_state_write(ctx.h, dev.h, j, a.ctypes.data_as(C.c_void_p), a.size))
    prev = state.prev_output
    if prev is not None:
        a = np.ascontiguousarray(_arr(prev))
        _lib.check(ctx.lib.fv_state_write(ctx.h, dev.h, -1, a.ctypes.data_as(C.c_void_p), a.size))
    return dev


def forward_full(net: WNetParams, sparse_input, state: RecurrentState, use_kernel_stage: bool = True):
    """Full pipeline with padding handled; returns (O, O_d, state') (network.py:296-323)."""
    import torch

    cfg = net.config
    x = sparse_input.dev if isinstance(sparse_input, DeviceTensor) else sparse_input
    if isinstance(x, torch.Tensor):
        xt = x.to(device="cuda", dtype=torch.float32)
    else:
        xt = torch.as_tensor(np.asarray(getattr(x, "data", x), dtype=np.float32), device="cuda")
    if xt.ndim != 4:
        raise ValueError(f"input must be (N, C, H, W), got {tuple(xt.shape)}")
    n, c, h, w = xt.shape
    if state.film_dims != (h, w):
        raise ValueError(f"carried state is for {state.film_dims}, input is {(h, w)}; reset the state")
    expect = 4 + (1 if cfg.include_mask_channel else 0)
    if c != expect:
        raise ValueError(f"input has {c + (3 if cfg.recurrent else 0)} channels, expected {cfg.in_channels}")
    if n != 1:
        raise ValueError("the device path reconstructs one frame per call (batch 1)")
    ctx = _lib.context()
    handle = net.handle(ctx)
    dev = _bind_state(net, state, ctx, handle)
    xt = xt[0].contiguous()
    _lib.check(ctx.lib.fv_state_set_input(ctx.h, dev.h, _lib.ptr(xt), c))
    o = torch.empty((3, h, w), dtype=torch.float32, device="cuda")
    od = torch.empty((3, h, w), dtype=torch.float32, device="cuda")
    _lib.check(ctx.lib.fv_reconstruct(ctx.h, handle, dev.h, int(bool(use_kernel_stage)), None,
                                      _lib.ptr(o), _lib.ptr(od)))
    state._consumed = True
    new = RecurrentState(film_dims=(h, w), _dev=dev, _config=cfg)
    return DeviceTensor(o[None]), DeviceTensor(od[None]), new


def forward_D(net: WNetParams, x, state: RecurrentState):
    """Coarse reconstruction (network.py:203-254): returns (O_d, H_d list, state'). The input's
    spatial dims must already be divisible by config.divisor. The D network (with the recurrent
    concat) runs on the device; H_d are the decoder hidden states the state now carries."""
    cfg = net.config
    arr = x.dev if isinstance(x, DeviceTensor) else x
    shape = tuple(arr.shape)
    if len(shape) != 4:
        raise ValueError(f"input must be (N, C, H, W), got {shape}")
    h, w = int(shape[2]), int(shape[3])
    if h % cfg.divisor or w % cfg.divisor:
        raise ValueError(f"input {h}x{w} not divisible by {cfg.divisor}; pad upstream")
    if state.film_dims != (h, w):
        raise ValueError(f"carried state is for {state.film_dims}, input is {(h, w)}; reset the state")
    _, od, new = forward_full(net, x, state, use_kernel_stage=False)
    return od, new.hidden, new


class KernelField:
    """Per-block predicted filter logits (network.py:257-265); normalized() softmaxes over the taps.
    Both are computed on the device (fv_kfield_logits) from the block's decoder hidden state."""

    def __init__(self, net: WNetParams, block: int, hd, kernel_size: int):
        self._net, self._block, self._hd, self.kernel_size = net, block, hd, kernel_size
        self._logits = None

    def _run(self, normalize: bool) -> "DeviceTensor":
        import torch

        hd = _dev_f32(self._hd)
        c, h, w = int(hd.shape[1]), int(hd.shape[2]), int(hd.shape[3])
        out = torch.empty((1, 9, h, w), dtype=torch.float32, device="cuda")
        ctx = _lib.context()
        _lib.check(ctx.lib.fv_kfield_logits(ctx.h, self._net.handle(ctx), self._block, _lib.ptr(hd[0].contiguous()),
                                            c, h, w, int(normalize), _lib.ptr(out)))
        return DeviceTensor(out)

    @property
    def logits(self) -> "DeviceTensor":
        if self._logits is None:
            self._logits = self._run(False)
        return self._logits

    def normalized(self) -> "DeviceTensor":
        return self._run(True)


def _dev_f32(t):
    """A (1, C, h, w) float32 CUDA tensor view of a DeviceTensor / array."""
    import torch

    if isinstance(t, DeviceTensor):
        return t.dev.to(torch.float32) if t.dev is not None else torch.as_tensor(t.data, device="cuda")
    if isinstance(t, torch.Tensor):
        return t.to(device="cuda", dtype=torch.float32)
    return torch.as_tensor(np.asarray(getattr(t, "data", t), dtype=np.float32), device="cuda")


def predict_kernel_fields(net: WNetParams, h_d: list) -> list[KernelField]:
    """One KernelField per block from the decoder hidden state at its level (network.py:268-277)."""
    cfg = net.config
    levels = _block_levels(cfg)
    by_level = {cfg.n_enc - j: h_d[j] for j in range(cfg.n_dec)}
    return [KernelField(net, i, by_level[lv], cfg.predicted_kernel) for i, lv in enumerate(levels)]


def forward_K(net: WNetParams, h_d: list, o_d) -> "DeviceTensor":
    """Refinement (network.py:280-293): filter O_d through the U shape with the kernels predicted from
    H_d -- the K-stage convs (tensor cores) and filter passes of the fused reconstruction, run on a
    scratch state holding H_d (fv_forward_k)."""
    import torch

    od = _dev_f32(o_d)
    h, w = int(od.shape[2]), int(od.shape[3])
    ctx = _lib.context()
    handle = net.handle(ctx)
    dev = _DevState(ctx, handle, h, w)
    if (dev.Hp, dev.Wp) != (h, w):
        raise ValueError(f"O_d {h}x{w} not divisible by {net.config.divisor}; pad upstream")
    for j, t in enumerate(h_d):
        a = np.ascontiguousarray(_dev_f32(t).cpu().numpy())
        _lib.check(ctx.lib.fv_state_write(ctx.h, dev.h, j, a.ctypes.data_as(C.c_void_p), a.size))
    out = torch.empty((3, h, w), dtype=torch.float32, device="cuda")
    _lib.check(ctx.lib.fv_forward_k(ctx.h, handle, dev.h, _lib.ptr(od[0].contiguous()), _lib.ptr(out)))
    res = DeviceTensor(out[None])
    res._scratch = dev  # the scratch state lives until the result does (its kernels are stream-ordered)
    return res


def forward_sparse(net: WNetParams, rgba, bits, state: RecurrentState, use_kernel_stage: bool = True):
    """_reconstruct_frame (bench.py:166-175) on device buffers: the input packing x = rgba*m ++ m
    runs in fv_pack_input straight into the network's NHWC8 input, then the W-Net, and the clipped
    (H, W, 3) image is written by the output stage. rgba: (H, W, 4) float32 CUDA tensor; bits:
    (H, W) uint8 CUDA tensor. Returns (rgb (H, W, 3) CUDA tensor in [0, 1], O, O_d, state')."""
    import torch

    cfg = net.config
    if not cfg.include_mask_channel:
        raise ValueError("forward_sparse packs the mask channel; this network has none")
    h, w = int(rgba.shape[0]), int(rgba.shape[1])
    if state.film_dims != (h, w):
        raise ValueError(f"carried state is for {state.film_dims}, input is {(h, w)}; reset the state")
    ctx = _lib.context()
    handle = net.handle(ctx)
    dev = _bind_state(net, state, ctx, handle)
    rgba = rgba.to(device="cuda", dtype=torch.float32).contiguous()
    bits = bits.to(device="cuda", dtype=torch.uint8).contiguous()
    _lib.check(ctx.lib.fv_pack_input(ctx.h, dev.h, _lib.ptr(rgba), _lib.ptr(bits)))
    rgb = torch.empty((h, w, 3), dtype=torch.float32, device="cuda")
    o = torch.empty((3, h, w), dtype=torch.float32, device="cuda")
    od = torch.empty((3, h, w), dtype=torch.float32, device="cuda")
    _lib.check(ctx.lib.fv_reconstruct(ctx.h, handle, dev.h, int(bool(use_kernel_stage)), _lib.ptr(rgb),
                                      _lib.ptr(o), _lib.ptr(od)))
    state._consumed = True
    new = RecurrentState(film_dims=(h, w), _dev=dev, _config=cfg)
    return rgb, DeviceTensor(o[None]), DeviceTensor(od[None]), new


def detach_state(state: RecurrentState) -> RecurrentState:
    return state


_CKPT_MAGIC = b"FVRCKPT1"


def save_network(net: WNetParams, path, meta: dict | None = None) -> None:
    """FVRCKPT1: magic, u32 header length, JSON manifest, little-endian f32 payload."""
    meta = dict(meta or {})
    meta.update(block_config=net.config.to_string(), predicted_kernel=net.config.predicted_kernel,
                recurrent=net.config.recurrent, include_mask_channel=net.config.include_mask_channel)
    manifest, blobs = [], []
    for name, arr in net.named_arrays().items():
        a = np.ascontiguousarray(arr, dtype="<f4")
        manifest.append({"name": name, "shape": list(a.shape), "dtype": "float32"})
        blobs.append(a.tobytes())
    header = json.dumps({"version": 1, "params": manifest, "meta": meta}).encode()
    with open(path, "wb") as f:
        f.write(_CKPT_MAGIC)
        f.write(struct.pack("<I", len(header)))
        f.write(header)
        for b in blobs:
            f.write(b)


def load_network(path) -> tuple[WNetParams, dict]:
    blob = Path(path).read_bytes()
    if blob[:8] != _CKPT_MAGIC:
        raise ValueError(f"not a checkpoint file: {path}")
    (hlen,) = struct.unpack("<I", blob[8:12])
    header = json.loads(blob[12: 12 + hlen].decode())
    if header.get("version") != 1:
        raise ValueError(f"unsupported checkpoint version {header.get('version')}")
    meta = header.get("meta", {})
    config = NetConfig.from_string(meta["block_config"],
                                   predicted_kernel=int(meta.get("predicted_kernel", 3)),
                                   recurrent=bool(meta.get("recurrent", True)),
                                   include_mask_channel=bool(meta.get("include_mask_channel", True)))
    net = init_network(config, seed=0)
    off = 12 + hlen
    for entry in header["params"]:
        count = int(np.prod(entry["shape"])) if entry["shape"] else 1
        arr = np.frombuffer(blob[off: off + 4 * count], dtype="<f4").reshape(entry["shape"]).copy()
        off += 4 * count
        name = entry["name"]
        if name not in net.params:
            raise ValueError(f"checkpoint parameter {name!r} not in network")
        if net.params[name].shape != arr.shape:
            raise ValueError(f"checkpoint shape mismatch for {name!r}")
        net.params[name] = arr.astype(np.float32)
    return net, meta


def truncate_fp16(arr: np.ndarray) -> np.ndarray:
    """Binary16 storage round trip with clamping (autograd.py:499-503)."""
    return np.clip(arr, -65504.0, 65504.0).astype(np.float16).astype(arr.dtype)


def quantized_net(net: WNetParams, mode: str = "fp16") -> WNetParams:
    """bench._quantized_net (bench.py:304-315): conv weights stored at `mode`, biases fp32."""
    if mode not in ("fp32", "fp16"):
        raise ValueError(f"unsupported storage precision {mode!r}")
    params = {}
    for name, p in net.named_arrays().items():
        a = p.copy()
        if mode == "fp16" and name.endswith(".w"):
            a = truncate_fp16(a)
        params[name] = a
    return WNetParams(config=net.config, params=params)
