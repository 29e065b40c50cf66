"""ctypes binding of libfovnet.so (the C ABI declared in include/fovnet.h).

The library is the only compute path: nothing in this package falls back to the
CPU. Loading fails loudly when the shared object is missing, and every context
creation fails loudly when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# FV_LIBFOVNET: alternative build of the same library (A/B runs of tools/probes; never set in tests)
LIB_PATH = Path(os.environ["FV_LIBFOVNET"]) if os.environ.get("FV_LIBFOVNET") else _HERE / "libfovnet.so"

FV_E_INVALID = -1
FV_E_CUDA = -2
FV_E_NOMEM = -3
FV_E_STATE = -4
FV_E_UNSUPPORTED = -5

# kernel classes of fv_ctx_kernel_time (include/fovnet.h)
FV_KC_MASK, FV_KC_MARCH_MAIN, FV_KC_MARCH_SHADOW, FV_KC_MARCH_COMPOSITE, FV_KC_CONV, FV_KC_NETOPS, FV_KC_OTHER = range(7)
KERNEL_CLASSES = {"mask": FV_KC_MASK, "march_main": FV_KC_MARCH_MAIN, "march_shadow": FV_KC_MARCH_SHADOW,
                  "march_composite": FV_KC_MARCH_COMPOSITE, "conv": FV_KC_CONV, "netops": FV_KC_NETOPS,
                  "other": FV_KC_OTHER}

LIGHT_NONE, LIGHT_DIRECTIONAL, LIGHT_POINT = 0, 1, 2
PREC_FP32, PREC_FP64, PREC_FP32_STRICT = 0, 1, 2


class FvCamera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("look_at", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_y", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class FvLight(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("vec", C.c_double * 3),
                ("intensity", C.c_double * 3)]


class FvSettings(C.Structure):
    _fields_ = [("step_size", C.c_double), ("shadow_step_factor", C.c_double),
                ("early_term_alpha", C.c_double), ("background", C.c_double * 4),
                ("ambient", C.c_double), ("reference_step", C.c_double),
                ("shadow_min_transmittance", C.c_double), ("precision", C.c_int32),
                ("_pad", C.c_int32)]


class FvFovea(C.Structure):
    _fields_ = [("focus", C.c_double * 2), ("sigma", C.c_double), ("base_density", C.c_double),
                ("pixel_scale", C.c_double)]


class FvStats(C.Structure):
    _fields_ = [("rays", C.c_uint64), ("hit_rays", C.c_uint64), ("samples_main", C.c_uint64),
                ("samples_shadow", C.c_uint64)]


P = C.c_void_p
I = C.c_int
I64 = C.c_int64
D = C.c_double
_SIGS = {
    "fv_last_error": (C.c_char_p, []),
    "fv_version": (I, []),
    "fv_ctx_create": (I, [I, C.POINTER(P)]),
    "fv_ctx_destroy": (I, [P]),
    "fv_ctx_set_stream": (I, [P, P]),
    "fv_ctx_stream": (P, [P]),
    "fv_sync": (I, [P]),
    "fv_noise_upload": (I, [P, P, I, I, I]),
    "fv_stats_read": (I, [P, C.POINTER(FvStats)]),
    "fv_stats_reset": (I, [P]),
    "fv_launch_count": (C.c_uint64, [P]),
    "fv_ctx_set_kernel_timing": (I, [P, I]),
    "fv_ctx_kernel_time": (I, [P, I, C.POINTER(D), C.POINTER(D), C.POINTER(C.c_uint64)]),
    "fv_mask_compact": (I, [P, I, I, I, C.POINTER(FvFovea), P, P, P, P, P]),
    "fv_mask_compact_tau": (I, [P, I, I, I, P, P, P, P, P]),
    "fv_tau_map": (I, [P, I, I, C.POINTER(FvFovea), P, P]),
    "fv_volume_create": (I, [P, I, I, I, C.POINTER(D), C.POINTER(P)]),
    "fv_volume_wrap": (I, [P, I, I, I, C.POINTER(D), P, C.POINTER(P)]),
    "fv_volume_destroy": (I, [P]),
    "fv_volume_upload": (I, [P, P, P, I]),
    "fv_volume_procedural": (I, [P, P, I, C.POINTER(D)]),
    "fv_volume_from_raw": (I, [P, P, P, I, C.POINTER(D), C.POINTER(I64)]),
    "fv_volume_set_tf": (I, [P, P, P, I]),
    "fv_volume_data": (P, [P]),
    "fv_render_sparse": (I, [P, P, C.POINTER(FvCamera), C.POINTER(FvLight), C.POINTER(FvSettings),
                             P, P, I, P, P, P, C.POINTER(FvStats)]),
    "fv_render_full": (I, [P, P, C.POINTER(FvCamera), C.POINTER(FvLight), C.POINTER(FvSettings),
                           P, P, C.POINTER(FvStats)]),
    "fv_shard_rays": (I, [P, P, P, I, I, I, P, P]),
    "fv_pack_records": (I, [P, P, P, P, I, P, P]),
    "fv_scatter_records": (I, [P, P, P, P, I64, I, P]),
    "fv_pack_rgb8": (I, [P, P, I, I, I64, I64, I64, P]),
    "fv_metric_sqdiff": (I, [P, P, P, P, P, I, I, I, I, C.POINTER(D)]),
    "fv_metric_ssim": (I, [P, P, P, I, I, I, I, I, I, C.POINTER(D), C.POINTER(D)]),
    "fv_render_sparse_naive": (I, [P, P, C.POINTER(FvCamera), C.POINTER(FvLight), C.POINTER(FvSettings),
                                   P, P, P, P, P, C.POINTER(FvStats)]),
    "fv_net_create": (I, [P, C.c_char_p, I, I, I, C.POINTER(P)]),
    "fv_net_destroy": (I, [P]),
    "fv_net_set_param": (I, [P, P, C.c_char_p, P, I64]),
    "fv_state_create": (I, [P, P, I, I, C.POINTER(P)]),
    "fv_state_reset": (I, [P, P]),
    "fv_state_destroy": (I, [P]),
    "fv_state_net_input": (P, [P]),
    "fv_state_dims": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
    "fv_pack_input": (I, [P, P, P, P]),
    "fv_state_set_input": (I, [P, P, P, I]),
    "fv_reconstruct": (I, [P, P, P, I, P, P, P]),
    "fv_state_read": (I, [P, P, I, P, I64, C.POINTER(I64)]),
    "fv_state_write": (I, [P, P, I, P, I64]),
    "fv_debug_conv3x3": (I, [P, I, I, I, I, P, P, P, P, P, I]),
    "fv_frame": (I, [P, P, P, P, C.POINTER(FvCamera), C.POINTER(FvLight), C.POINTER(FvSettings),
                     C.POINTER(FvFovea), I, P, C.POINTER(D)]),
    "fv_frames": (I, [P, P, P, P, I, C.POINTER(FvCamera), C.POINTER(FvLight), C.POINTER(FvSettings),
                      C.POINTER(FvFovea), C.POINTER(I), C.POINTER(P)]),
    "fv_forward_k": (I, [P, P, P, P, P]),
    "fv_kfield_logits": (I, [P, P, I, P, I, I, I, I, P]),
    "fv_generate_rays": (I, [P, C.POINTER(FvCamera), P, P, I64, P, P]),
    "fv_sample_trilinear": (I, [P, P, P, I64, P]),
    "fv_tf_apply": (I, [P, P, I, P, I64, P]),
    "fv_tile_field": (I, [P, I, I, I, P]),
    "fv_tau_sum": (I, [P, I, I, C.POINTER(FvFovea), P, P, P]),
    "fv_foveal_density": (I, [P, P, P, I64, D, D, P]),
    "fv_direct_draws": (I, [P, I, I, C.POINTER(FvFovea), P, P, P, I64, P]),
    "fv_pack_records16": (I, [P, P, P, P, I, P]),
    "fv_scatter_records16": (I, [P, P, P, I64, I, I]),
    "fv_window_input": (I, [P, P, P, I, I, I]),
    "fv_state_band": (I, [P, P, I, I, I, P, C.POINTER(I64)]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load libfovnet.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class FvError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().fv_last_error().decode(errors="replace")
    if rc in (FV_E_INVALID, FV_E_STATE):
        raise ValueError(msg)
    raise FvError(f"libfovnet error {rc}: {msg}")


def ptr(t) -> C.c_void_p | None:
    """Device pointer of a torch tensor (None stays NULL)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


class Context:
    """One fv_ctx bound to a device and to torch's current stream on that device."""

    def __init__(self, device: int = 0, stream=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("libfovnet needs a CUDA (sm_100a) device; none is available")
        self.lib = load()
        self.device = device
        h = C.c_void_p()
        check(self.lib.fv_ctx_create(device, C.byref(h)))
        self.h = h
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        check(self.lib.fv_ctx_set_stream(self.h, C.c_void_p(self.stream.cuda_stream)))
        self.noise_key = None

    def sync(self) -> None:
        check(self.lib.fv_sync(self.h))

    def launches(self) -> int:
        return int(self.lib.fv_launch_count(self.h))

    def stats(self) -> FvStats:
        s = FvStats()
        check(self.lib.fv_stats_read(self.h, C.byref(s)))
        return s

    def reset_stats(self) -> None:
        check(self.lib.fv_stats_reset(self.h))

    def set_kernel_timing(self, enable: bool) -> None:
        """Bracket every library launch with CUDA events (totals reset on each call)."""
        check(self.lib.fv_ctx_set_kernel_timing(self.h, 1 if enable else 0))

    def kernel_time(self, kernel_class: int) -> tuple[float, float, int]:
        """(summed launch ms, summed algorithmic work, launches) of one FV_KC_* class."""
        ms, work, n = C.c_double(), C.c_double(), C.c_uint64()
        check(self.lib.fv_ctx_kernel_time(self.h, kernel_class, C.byref(ms), C.byref(work), C.byref(n)))
        return ms.value, work.value, int(n.value)

    def ensure_noise(self, stack) -> None:
        """Upload a NoiseStack once per context (keyed by object identity + shape)."""
        key = (id(stack), stack.values.shape)
        if self.noise_key == key:
            return
        import numpy as np

        vals = np.ascontiguousarray(stack.values, dtype="<f4")
        t, h, w = vals.shape
        check(self.lib.fv_noise_upload(self.h, vals.ctypes.data_as(C.c_void_p), t, h, w))
        self.noise_key = key
        self._noise_ref = stack

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and _lib is not None:
                _lib.fv_ctx_destroy(self.h)
        except Exception:
            pass


_ctx_local = threading.local()


def context(device: int | None = None) -> Context:
    """Per-thread default context (one CUDA stream per thread, as the viewer's executor needs)."""
    import torch

    dev = torch.cuda.current_device() if device is None else device
    cache = getattr(_ctx_local, "ctx", None)
    if cache is None:
        cache = _ctx_local.ctx = {}
    if dev not in cache:
        cache[dev] = Context(dev)
    return cache[dev]


def lib_path() -> str:
    return os.fspath(LIB_PATH)
