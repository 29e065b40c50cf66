"""Viewer caller of the hot path (reference viewer.py:161-223): render_frame's device path against
the messages the reference produced (tests/golden/viewer_small.npz, made by make_golden.gen_viewer)."""
import io
import struct
from dataclasses import dataclass, replace

import numpy as np
import pytest

from paper_2209_09965_b200 import viewer as V
from paper_2209_09965_b200.sample_maps import FAST_PRESET, FoveaConfig, pixel_scale_for_film


@dataclass
class Session:
    """The attributes render_frame reads from the caller's session (reference SessionState)."""

    fovea: FoveaConfig
    mode: str = "sparse_raw"
    frame_idx: int = 0
    recurrent: object = None
    warning: str = ""


def viewer_fovea(w, h, focus=None, p_b=FAST_PRESET["base_density"], sigma=FAST_PRESET["sigma"]):
    # the reference viewer's fovea: film-centre focus, fast preset, pixel scale at fraction 0.25
    return FoveaConfig(focus=focus if focus is not None else ((w - 1) / 2.0, (h - 1) / 2.0), sigma=sigma,
                       base_density=p_b, pixel_scale=pixel_scale_for_film((h, w), fraction=0.25))


def test_header_layout():
    hdr = struct.pack(V.HEADER_FMT, 7, 64, 36, 2, 1, 1.5, 2.5, 3.5, 7.5, 10.0, 20.0, 0.03, 0.02, 10)
    assert len(hdr) == 46 and V.MODES[2] == "ground_truth"


@pytest.mark.gpu
def test_render_frame_every_mode_vs_reference_messages(golden):
    from PIL import Image

    from paper_2209_09965_b200 import network as N
    from paper_2209_09965_b200.noise import default_stack
    from paper_2209_09965_b200.renderer import RenderSettings, Scene
    from paper_2209_09965_b200.volume import Camera, Light, TransferFunction, make_procedural_volume

    g = np.load(golden / "viewer_small.npz")
    vol = make_procedural_volume("sphere_shells", (32, 32, 32))
    scene = Scene(volume=vol, tf=TransferFunction.default(),
                  light=Light(direction=(-1.0, -1.0, -0.5), intensity=(1.0, 1.0, 1.0)))
    net = N.quantized_net(N.init_network(N.NetConfig.from_string(N.DESK_BLOCKS), seed=7), "fp16")
    cam = Camera(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0, width=64, height=36)
    svc = V.RenderService(scene, film=(64, 36), checkpoint=net, noise=default_stack(),
                          settings=RenderSettings(step_size=1.0), camera=cam)
    # the reference's control plan (make_golden.gen_viewer): fovea changes persist across frames
    plan = [("sparse_raw", viewer_fovea(64, 36)), ("reconstructed", viewer_fovea(64, 36)),
            ("reconstructed", viewer_fovea(64, 36, focus=(10.0, 30.0), p_b=0.2)),
            ("ground_truth", viewer_fovea(64, 36, focus=(10.0, 30.0), p_b=0.2)),
            ("side_by_side", viewer_fovea(64, 36, focus=(10.0, 30.0), p_b=0.2, sigma=0.5))]
    state = Session(fovea=plan[0][1])
    for i, (mode, fovea) in enumerate(plan):
        state = replace(state, mode=mode, fovea=fovea)
        blob, state = svc.render_frame(state)
        fields = struct.unpack(V.HEADER_FMT, blob[:46])
        png = blob[46:46 + fields[-1]]
        img = np.asarray(Image.open(io.BytesIO(png)))
        ref = g[f"img{i}"]
        assert img.shape == ref.shape, (i, img.shape)
        hdr = np.array([fields[0], fields[1], fields[2], fields[3], fields[9], fields[10], fields[11], fields[12]],
                       dtype=np.float64)
        assert np.array_equal(hdr, g[f"hdr{i}"].astype(np.float32).astype(np.float64)), (i, hdr, g[f"hdr{i}"])
        diff = np.abs(img.astype(int) - ref.astype(int))
        assert diff.max() <= 2 and (diff <= 1).mean() >= 0.99, (i, diff.max(), (diff <= 1).mean())
    assert state.frame_idx == len(plan)
