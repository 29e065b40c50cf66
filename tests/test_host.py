"""CPU-only checks of the boundary and the host-side mirror of the reference API."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "fovnet.h").read_text()
    return sorted(set(re.findall(r"FV_API\s+[\w\s\*]+?\b(fv_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2209_09965_b200 import _lib

    if not _lib.LIB_PATH.exists():
        import __graft_entry__

        __graft_entry__.build()
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.fv_version() == 1


def test_context_fails_loudly_without_gpu():
    import torch

    from paper_2209_09965_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        _lib.Context(0)


def test_fovea_config_validation():
    from paper_2209_09965_b200.sample_maps import FoveaConfig

    with pytest.raises(ValueError, match=">= 0"):
        FoveaConfig(focus=(0, 0), sigma=-1.0)
    with pytest.raises(ValueError, match="finite"):
        FoveaConfig(focus=(np.inf, 0))
    with pytest.raises(ValueError, match=r"\[0,1\]"):
        FoveaConfig(focus=(0, 0), base_density=1.5)


def test_pixel_scale_matches_default_at_720p():
    from paper_2209_09965_b200.sample_maps import pixel_scale_for_film

    assert pixel_scale_for_film((720, 1280)) == pytest.approx(1.0 / 32.0, rel=2e-2)
    assert pixel_scale_for_film((1080, 1920)) == pytest.approx(0.02058, rel=1e-3)


def test_netconfig_validation_and_layout():
    from paper_2209_09965_b200.network import FULL_BLOCKS, NetConfig, _conv_channels

    cfg = NetConfig.from_string(FULL_BLOCKS)
    assert cfg.n_enc == 3 and cfg.n_dec == 4 and cfg.divisor == 8 and cfg.in_channels == 8
    blocks, k_in = _conv_channels(cfg)
    assert blocks == [(8, 64), (64, 64), (64, 80), (176, 96), (256, 80), (208, 64), (192, 64)]
    assert k_in == [64, 64, 80, 96, 80, 64, 64]
    with pytest.raises(ValueError, match="one more"):
        NetConfig.from_string("e16-e16-d24-d24")
    with pytest.raises(ValueError, match="e-blocks then d-blocks"):
        NetConfig.from_string("e16-d24-e16-d24-d16")
    with pytest.raises(ValueError, match="bad block token"):
        NetConfig.from_string("x16-d24")


def test_init_network_matches_oracle_weights():
    from oracle import fovray_oracle as O
    from paper_2209_09965_b200.network import DESK_BLOCKS, NetConfig, init_network

    net = init_network(NetConfig.from_string(DESK_BLOCKS), seed=7)
    ref = O.init_params(DESK_BLOCKS, 7)
    assert set(net.params) == set(ref)
    for k in ref:
        assert np.array_equal(net.params[k], ref[k]), k


def test_checkpoint_roundtrip(tmp_path):
    from paper_2209_09965_b200.network import DESK_BLOCKS, NetConfig, init_network, load_network, save_network

    net = init_network(NetConfig.from_string(DESK_BLOCKS), seed=3)
    save_network(net, tmp_path / "n.ckpt", meta={"note": "x"})
    back, meta = load_network(tmp_path / "n.ckpt")
    assert meta["note"] == "x" and back.config == net.config
    for k, v in net.params.items():
        assert np.array_equal(back.params[k], v)


def test_checkpoint_format_is_reference_fvrckpt1(tmp_path):
    from paper_2209_09965_b200.network import DESK_BLOCKS, NetConfig, init_network, save_network

    save_network(init_network(NetConfig.from_string(DESK_BLOCKS), seed=1), tmp_path / "n.ckpt")
    assert (tmp_path / "n.ckpt").read_bytes()[:8] == b"FVRCKPT1"


def test_noise_stack_roundtrip_and_validation(tmp_path, stack_values):
    from paper_2209_09965_b200.noise import NoiseStack, default_stack, load_stack, save_stack

    st = default_stack()
    assert np.array_equal(st.values, stack_values)
    save_stack(st, tmp_path / "s.noise")
    assert np.array_equal(load_stack(tmp_path / "s.noise").values, st.values)
    bad = st.values.copy()
    bad[0, 0, 0] = bad[0, 0, 1]
    with pytest.raises(ValueError, match="rank permutation"):
        NoiseStack(values=bad)


def test_orbit_cameras_match_oracle():
    from oracle import fovray_oracle as O
    from paper_2209_09965_b200.renderer import OrbitPathSpec
    from paper_2209_09965_b200.volume import Camera

    spec = OrbitPathSpec(n_frames=500)
    dims = (512, 512, 512)
    ext = np.asarray(dims, float)

    class V:  # host-only stand-in for VolumeGrid geometry
        extent = ext

        @staticmethod
        def center():
            return ext * 0.5

    from paper_2209_09965_b200.renderer import orbit_cameras

    cams = orbit_cameras(spec, V, 1920, 1080)
    for i in (0, 1, 250, 499):
        pos, look = O.orbit_camera(i, 500, dims)
        assert cams[i].position == pos and cams[i].look_at == look
    assert isinstance(cams[0], Camera)


def test_camera_and_light_validation():
    from paper_2209_09965_b200.volume import Camera, Light, TransferFunction

    with pytest.raises(ValueError, match="fov_y"):
        Camera(position=(0, 0, 0), look_at=(1, 0, 0), fov_y=0.0)
    with pytest.raises(ValueError, match="coincide"):
        Camera(position=(1, 1, 1), look_at=(1, 1, 1))
    with pytest.raises(ValueError, match="parallel"):
        Camera(position=(0, 0, 0), look_at=(0, 1, 0))
    with pytest.raises(ValueError, match="exactly one"):
        Light()
    with pytest.raises(ValueError, match=r"\[0,1\]"):
        TransferFunction(lut=np.full((2, 4), 2.0))
    assert TransferFunction.default().lut.shape == (7, 4)


def test_render_settings_validation():
    from paper_2209_09965_b200.renderer import RenderSettings

    with pytest.raises(ValueError):
        RenderSettings(step_size=0.0)
    with pytest.raises(ValueError):
        RenderSettings(shadow_step_factor=0.5)
    with pytest.raises(ValueError):
        RenderSettings(precision="fp8")
    s = RenderSettings().c_struct()
    assert s.precision == 0 and s.shadow_step_factor == 4.0
