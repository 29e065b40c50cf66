"""Viewer caller of the hot path (viewer.py:50-242): control handling and frame messages (CPU),
render_frame against messages the reference produced (GPU)."""
import io
import struct

import numpy as np
import pytest

from paper_2209_09965_b200 import viewer as V


def test_handle_control_clamps_and_warnings():
    st = V.default_session((64, 36))
    assert st.fovea.focus == (31.5, 17.5) and st.mode == "sparse_raw"
    s2 = V.handle_control(st, {"type": "control", "focus": [-3, 50], "p_b": 5.0, "sigma": -1, "mode": "bogus",
                               "extra": 1}, (64, 36), has_checkpoint=False)
    assert s2.fovea.focus == (0.0, 35.0) and s2.fovea.base_density == 1.0 and s2.fovea.sigma == 0.0
    assert s2.mode == "sparse_raw"
    assert s2.warning == ("ignored unknown field 'extra'; focus clamped to film bounds; p_b clamped; "
                          "sigma clamped; unknown mode 'bogus'")
    s3 = V.handle_control(st, {"mode": "reconstructed"}, (64, 36), has_checkpoint=False)
    assert s3.mode == "sparse_raw" and "no checkpoint" in s3.warning
    s4 = V.handle_control(st, {"mode": "side_by_side", "p_b": 0.5}, (64, 36), has_checkpoint=True)
    assert s4.mode == "side_by_side" and s4.fovea.base_density == 0.5 and s4.warning == ""


def test_frame_message_layout_round_trip():
    png = b"\x89PNG-bytes"
    hdr = struct.pack(V.HEADER_FMT, 7, 64, 36, 2, 1, 1.5, 2.5, 3.5, 7.5, 10.0, 20.0, 0.03, 0.02, len(png))
    d = V.parse_frame_message(hdr + png + "careful".encode())
    assert V.HEADER_SIZE == 46
    assert d["frame_id"] == 7 and (d["width"], d["height"]) == (64, 36) and d["mode"] == "ground_truth"
    assert d["png"] == png and d["warning"] == "careful"
    assert d["timings"]["total_ms"] == 7.5 and d["focus"] == (10.0, 20.0)


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
    state = V.default_session((64, 36))
    plan = [("sparse_raw", {}), ("reconstructed", {}), ("reconstructed", {"focus": [10.0, 30.0], "p_b": 0.2}),
            ("ground_truth", {}), ("side_by_side", {"sigma": 0.5})]
    for i, (mode, ctl) in enumerate(plan):
        state = V.handle_control(state, dict(ctl, mode=mode), svc.film, has_checkpoint=True)
        blob, state = svc.render_frame(state)
        d = V.parse_frame_message(blob)
        img = np.asarray(Image.open(io.BytesIO(d["png"])))
        ref = g[f"img{i}"]
        assert img.shape == ref.shape, (i, img.shape)
        hdr = np.array([d["frame_id"], d["width"], d["height"], V.MODES.index(d["mode"]), d["focus"][0],
                        d["focus"][1], d["p_b"], d["sigma"]], dtype=np.float64)
        assert np.array_equal(hdr, g[f"hdr{i}"]), (i, hdr, g[f"hdr{i}"])
        diff = np.abs(img.astype(int) - ref.astype(int))
        assert diff.max() <= 2 and (diff <= 1).mean() >= 0.99, (i, diff.max(), (diff <= 1).mean())
    assert state.frame_idx == len(plan)
