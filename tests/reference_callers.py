"""The reference's own caller of the hot-path modules, run unchanged against this package.

`render_flythrough` below is the reference's function body (pkg/src/fovray/renderer.py:385-432,
verbatim) with only its two package-relative imports pointed at paper_2209_09965_b200 -- test
infrastructure (SURVEY.md 8(b) "callers unchanged"): tests/test_boundary.py runs it with the
device-backed modules swapped in and compares its frames with the package's own render_flythrough.
"""
import time

import numpy as np

from paper_2209_09965_b200.renderer import (RenderSettings, Scene, render_full, render_sparse_compact,
                                           render_sparse_direct, render_sparse_naive)
from paper_2209_09965_b200.volume import Camera


def render_flythrough(scene: Scene, cams: list[Camera],
                      settings: RenderSettings = RenderSettings(), mode: str = "full",
                      noise=None, fovea=None, rng: np.random.Generator | None = None):
    """Render a camera path; returns (frames, timing rows).

    Timing rows are (frame, mask_ms, render_ms, reconstruct_ms,
    total_ms); the noise frame index advances with the path frame.
    """
    from paper_2209_09965_b200.sample_maps import build_sample_mask, build_tau_map, c_max, compact_mask, draw_direct_samples

    if not cams:
        raise ValueError("camera path must have at least one frame")
    if mode not in ("full", "naive", "compact", "direct"):
        raise ValueError(f"unknown flythrough mode {mode!r}")
    if mode != "full" and (noise is None or fovea is None):
        raise ValueError(f"mode {mode!r} needs a noise stack and a fovea config")
    frames = []
    rows = []
    rng = rng if rng is not None else np.random.default_rng(0)
    for i, cam in enumerate(cams):
        if mode == "full":
            fr = render_full(scene, cam, settings)
        else:
            tic = time.perf_counter()
            cfg = fovea
            tau = build_tau_map(cfg, (cam.height, cam.width))
            if mode == "direct":
                count = max(1, int(round(c_max(tau) * cam.height * cam.width)))
                from paper_2209_09965_b200.noise import tile_field

                nf = tile_field(noise, cam.height, cam.width, i)
                work = draw_direct_samples(cfg, nf, count, rng)
            else:
                mask = build_sample_mask(noise, i, tau)
                if mode == "compact":
                    work = compact_mask(mask)
            mask_ms = (time.perf_counter() - tic) * 1e3
            if mode == "naive":
                fr = render_sparse_naive(scene, cam, mask, settings)
            elif mode == "compact":
                fr = render_sparse_compact(scene, cam, work, settings)
            else:
                fr = render_sparse_direct(scene, cam, work, settings)
            fr.mask_ms = mask_ms
            fr.total_ms = fr.mask_ms + fr.render_ms
        frames.append(fr)
        rows.append((i, fr.mask_ms, fr.render_ms, fr.reconstruct_ms, fr.total_ms))
    return frames, rows
