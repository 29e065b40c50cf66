"""Time the tcgen05 conv engine on synthetic NC8HW8 inputs through fv_debug_conv3x3 (kernel-timing
events around the conv launch only). usage: python tools/probes/conv_bench.py"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_09965_b200 import _lib  # noqa: E402

ctx = _lib.context()
SHAPES = [(8, 64, 1080, 1920), (64, 64, 1080, 1920), (192, 64, 1080, 1920), (64, 64, 540, 960),
          (208, 64, 540, 960), (256, 80, 270, 480), (192, 64, 270, 480), (176, 96, 135, 240), (64, 32, 1080, 1920)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]]
rng = np.random.default_rng(0)
for cin, cout, h, w in SHAPES:
    x = (torch.rand((cin // 8, h, w, 8), device="cuda", dtype=torch.float32) - 0.5).half()
    y = torch.empty((cout // 8, h, w, 8), device="cuda", dtype=torch.float16)
    wt = (rng.standard_normal((cout, cin, 3, 3)) * 0.05).astype(np.float32)
    b = np.zeros(cout, np.float32)
    args = (ctx.h, cin, cout, h, w, _lib.ptr(x), wt.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
            _lib.ptr(y), None, 1)
    for _ in range(3):
        _lib.check(ctx.lib.fv_debug_conv3x3(*args))
    ctx.set_kernel_timing(True)
    reps = 10
    for _ in range(reps):
        _lib.check(ctx.lib.fv_debug_conv3x3(*args))
    ms, flops, n = ctx.kernel_time(_lib.FV_KC_CONV)
    ctx.set_kernel_timing(False)
    us = ms / n * 1e3
    byts = (cin + cout) * h * w * 2
    print(f"{cin:4d}->{cout:3d} {h:5d}x{w:5d}: {us:8.1f} us  {flops / (ms / 1e3) / 1e12:7.1f} TFLOP/s  "
          f"{byts / (us / 1e6) / 1e9:7.0f} GB/s (in+out)")
