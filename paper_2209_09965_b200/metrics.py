"""Image and video quality metrics on the GPU: PSNR, SSIM, MS-SSIM and tPSNR (metrics.py:1-197).

Same definitions and edge behaviour as the reference: PSNR jointly over RGB with the 100 dB
sentinel for identical frames; SSIM on Rec.601 luma with an 11x11 Gaussian window (sigma 1.5,
K1=0.01, K2=0.03) averaged over valid window positions; MS-SSIM with the 5-scale weights
renormalised to the usable scales and contrast-structure means clamped at zero; tPSNR as PSNR of
(d+1)/2 temporal differences. Arithmetic is fp64 in libfovnet's metric kernels (csrc/metrics.cu);
inputs may be NumPy arrays or CUDA tensors of shape (H, W, C) (C >= 3) or (H, W) luma.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

PSNR_CAP_DB = 100.0
MSSSIM_WEIGHTS = (0.0448, 0.2856, 0.3001, 0.2363, 0.1333)
_SSIM_WINDOW = 11


def _dev(img):
    """(H, W, C) float64 contiguous CUDA tensor (fp32 inputs convert exactly)."""
    import torch

    t = img if isinstance(img, torch.Tensor) else torch.as_tensor(np.asarray(img))
    t = t.to(device="cuda", dtype=torch.float64)
    if t.dim() == 2:
        t = t.unsqueeze(-1)
    if t.dim() != 3:
        raise ValueError(f"images must be (H, W) or (H, W, C), got shape {tuple(t.shape)}")
    return t.contiguous()


def _hw(t) -> tuple[int, int]:
    return int(t.shape[0]), int(t.shape[1])


def _rgb_check(a, b, name):
    if a.shape[2] < 3 or b.shape[2] < 3:
        raise ValueError(f"{name} needs RGB images (C >= 3)")
    if _hw(a) != _hw(b):
        raise ValueError(f"{name} dims differ: {tuple(a.shape)} vs {tuple(b.shape)}")


def _from_mse(mse: float, peak: float) -> float:
    if mse == 0.0:
        return PSNR_CAP_DB
    return min(10.0 * float(np.log10(peak * peak / mse)), PSNR_CAP_DB)


def psnr(a, b, peak: float = 1.0) -> float:
    """10 log10(peak^2 / MSE) over RGB, capped at 100 dB for identity (metrics.py:40-49)."""
    ta, tb = _dev(a), _dev(b)
    _rgb_check(ta, tb, "psnr")
    h, w = _hw(ta)
    ctx = _lib.context()
    s = C.c_double()
    _lib.check(ctx.lib.fv_metric_sqdiff(ctx.h, _lib.ptr(ta), _lib.ptr(tb), None, None, h, w, int(ta.shape[2]),
                                        int(tb.shape[2]), C.byref(s)))
    return _from_mse(s.value / (h * w * 3), peak)


def _ssim_call(a, b, mode: int, scales: int = 0, weights=None) -> float:
    ta, tb = _dev(a), _dev(b)
    if _hw(ta) != _hw(tb):
        raise ValueError(f"{'ssim' if mode == 0 else 'msssim'} dims differ: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    h, w = _hw(ta)
    if min(h, w) < _SSIM_WINDOW:
        raise ValueError(f"frames smaller than the {_SSIM_WINDOW}px SSIM window: {(h, w)}")
    ctx = _lib.context()
    out = C.c_double()
    wts = (C.c_double * max(scales, 1))(*(weights if weights is not None else [0.0]))
    _lib.check(ctx.lib.fv_metric_ssim(ctx.h, _lib.ptr(ta), _lib.ptr(tb), h, w, int(ta.shape[2]), int(tb.shape[2]),
                                      mode, scales, wts, C.byref(out)))
    return float(out.value)


def ssim(a, b) -> float:
    """Mean SSIM over valid 11x11 Gaussian windows on Rec.601 luma (metrics.py:74-87)."""
    return _ssim_call(a, b, 0)


def msssim_scale_count(dims: tuple[int, int]) -> int:
    """Scales usable before the coarsest image drops under the SSIM window (metrics.py:96-102)."""
    m = 1
    size = min(dims)
    while m < len(MSSSIM_WEIGHTS) and size // 2 >= _SSIM_WINDOW:
        size //= 2
        m += 1
    return m


def msssim(a, b) -> float:
    """Multi-scale SSIM with automatic scale reduction and renormalised weights (metrics.py:104-130)."""
    ta = _dev(a)
    m = msssim_scale_count(_hw(ta))
    wts = np.asarray(MSSSIM_WEIGHTS[:m])
    wts = wts / wts.sum()
    return _ssim_call(ta, b, 1, m, [float(x) for x in wts])


def tpsnr(seq_a, seq_b) -> np.ndarray:
    """PSNR of temporal finite differences, one value per frame from 1 on (metrics.py:133-148)."""
    t = len(seq_a)
    if len(seq_b) != t:
        raise ValueError(f"sequence lengths differ: {t} vs {len(seq_b)}")
    if t < 2:
        raise ValueError(f"tpsnr needs at least 2 frames, got {t}")
    ctx = _lib.context()
    out = np.empty(t - 1)
    da = [_dev(x) for x in seq_a]
    db = [_dev(x) for x in seq_b]
    for i in range(1, t):
        _rgb_check(da[i], db[i], "tpsnr")
        h, w = _hw(da[i])
        s = C.c_double()
        _lib.check(ctx.lib.fv_metric_sqdiff(ctx.h, _lib.ptr(da[i]), _lib.ptr(db[i]), _lib.ptr(da[i - 1]),
                                            _lib.ptr(db[i - 1]), h, w, int(da[i].shape[2]), int(db[i].shape[2]),
                                            C.byref(s)))
        out[i - 1] = _from_mse(s.value / (h * w * 3), 1.0)
    return out


@dataclass
class QualityReport:
    """Per-frame metrics for a clip; tpsnr is NaN for frame 0 (metrics.py:151-179)."""

    psnr: np.ndarray
    ssim: np.ndarray
    msssim: np.ndarray
    tpsnr: np.ndarray

    @property
    def n_frames(self) -> int:
        return len(self.psnr)

    def aggregates(self) -> dict[str, float]:
        out = {}
        for name in ("psnr", "ssim", "msssim", "tpsnr"):
            vals = getattr(self, name)
            finite = vals[np.isfinite(vals)]
            out[f"{name}_mean"] = float(finite.mean()) if finite.size else float("nan")
            out[f"{name}_min"] = float(finite.min()) if finite.size else float("nan")
        return out

    def csv_rows(self) -> list[tuple]:
        rows = []
        for i in range(self.n_frames):
            tp = "" if np.isnan(self.tpsnr[i]) else f"{self.tpsnr[i]:.6f}"
            rows.append((i, f"{self.psnr[i]:.6f}", f"{self.ssim[i]:.6f}", f"{self.msssim[i]:.6f}", tp))
        return rows


def build_quality_report(pred_seq, gt_seq) -> QualityReport:
    """Per-frame PSNR / SSIM / MS-SSIM and tPSNR of a predicted clip against ground truth
    (metrics.py:182-197)."""
    t = len(pred_seq)
    if len(gt_seq) != t:
        raise ValueError(f"sequence lengths differ: {t} vs {len(gt_seq)}")
    ps = np.array([psnr(pred_seq[i], gt_seq[i]) for i in range(t)])
    ss = np.array([ssim(pred_seq[i], gt_seq[i]) for i in range(t)])
    ms = np.array([msssim(pred_seq[i], gt_seq[i]) for i in range(t)])
    tp = np.full(t, np.nan)
    if t >= 2:
        tp[1:] = tpsnr(pred_seq, gt_seq)
    return QualityReport(psnr=ps, ssim=ss, msssim=ms, tpsnr=tp)
