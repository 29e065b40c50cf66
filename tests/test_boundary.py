"""The drop-in boundary beyond the frame loop: the reference's per-sample building
blocks and kernel-stage API as device calls, checked against reference-made goldens
(tests/golden/boundary_small.npz, make_golden.gen_boundary), and the reference's own caller
render_flythrough (tests/reference_callers.py, its body verbatim) run against this package.

Tolerances: fp64 building blocks 1e-12 (FMA contraction on the device); tile_field / tile_lookup
exact; forward_D / forward_K / K fields with the fp16 weights of the desk net against the fp32
reference: 2e-2 x max(1, |ref|) (the network tier's storage rounding, as test_gpu_parity).
"""
import numpy as np
import pytest

from oracle import fovray_oracle as O

CAM = dict(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0, width=64, height=36)


@pytest.fixture(scope="module")
def gb(golden):
    return np.load(golden / "boundary_small.npz")


# ---- CPU: the oracle restatements against the reference-made values
def test_oracle_building_blocks_vs_reference(gb, stack_values):
    o, d = O.generate_rays(CAM, gb["ray_us"], gb["ray_vs"])
    np.testing.assert_allclose(o, gb["ray_o"], rtol=0, atol=0)
    np.testing.assert_allclose(d, gb["ray_d"], rtol=0, atol=1e-15)
    vol, _ = O.procedural_volume("vortex_field", (33, 17, 9))
    np.testing.assert_allclose(O.sample_trilinear(vol, (1.0, 2.0, 0.5), gb["tri_pts"]), gb["tri_vals"], rtol=0,
                               atol=1e-14)
    np.testing.assert_allclose(O.tf_apply(O.DEFAULT_LUT, gb["tf_s"]), gb["tf_rgba"], rtol=0, atol=1e-15)
    assert np.array_equal(O.noise_field(stack_values, 70, 150, 11), gb["tile_field"])


# ---- GPU: the device-backed functions
gpu = pytest.mark.gpu


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@gpu
def test_noise_tile_field_and_lookup(gb):
    _torch()
    from paper_2209_09965_b200.noise import default_stack, tile_field, tile_lookup

    st = default_stack()
    assert np.array_equal(tile_field(st, 70, 150, 11), gb["tile_field"])
    got = [tile_lookup(st, u, v, f) for u, v, f in [(0, 0, 0), (70, 3, 9), (-3, 200, 13)]]
    assert np.array_equal(np.array(got), gb["tile_lookup"])


@gpu
def test_generate_rays_sample_trilinear_tf_apply(gb):
    _torch()
    from paper_2209_09965_b200.volume import (Camera, TransferFunction, generate_rays, make_procedural_volume,
                                              sample_trilinear)

    o, d = generate_rays(Camera(**CAM), gb["ray_us"], gb["ray_vs"])
    np.testing.assert_array_equal(o, gb["ray_o"])
    np.testing.assert_allclose(d, gb["ray_d"], rtol=0, atol=1e-15)
    vol = make_procedural_volume("vortex_field", (33, 17, 9), spacing=(1.0, 2.0, 0.5))
    np.testing.assert_allclose(sample_trilinear(vol, gb["tri_pts"]), gb["tri_vals"], rtol=0, atol=1e-12)
    assert sample_trilinear(vol, gb["tri_pts"][-1]) == pytest.approx(gb["tri_vals"][-1], abs=1e-12)
    np.testing.assert_allclose(TransferFunction.default().apply(gb["tf_s"]), gb["tf_rgba"], rtol=0, atol=1e-12)
    assert TransferFunction.default().apply(gb["tf_s"].reshape(2, -1)).shape == (2, gb["tf_s"].size // 2, 4)


@gpu
def test_foveal_density_and_c_max(gb):
    _torch()
    from paper_2209_09965_b200 import sample_maps as S

    dx = np.arange(-40, 41, dtype=np.float64)[None, :]
    dy = np.arange(-20, 21, dtype=np.float64)[:, None]
    np.testing.assert_allclose(S.foveal_density((dx, dy), 0.06, 0.02), gb["fovd"], rtol=2e-16, atol=0)
    assert S.foveal_density((3.0, 4.0), 0.06, 0.02) == pytest.approx(gb["fovd"][24, 43], rel=2e-16)
    cfg = S.FoveaConfig(focus=(959.5, 539.5), sigma=0.06, base_density=0.07,
                        pixel_scale=S.pixel_scale_for_film((1080, 1920)))
    ref = O.tau_map(1080, 1920, cfg.focus, 0.06, 0.07, cfg.pixel_scale)
    import math

    assert S.c_max(S.build_tau_map(cfg, (1080, 1920))) == pytest.approx(math.fsum(ref.ravel()) / ref.size, rel=1e-12)


@gpu
def test_kernel_stage_split_api_vs_reference(gb):
    _torch()
    from paper_2209_09965_b200 import network as N

    net = N.init_network(N.NetConfig.from_string(N.DESK_BLOCKS), seed=5)
    state = N.reset_state(net.config, (32, 48))

    def close(got, ref, what):
        assert np.abs(got - ref).max() <= 2e-2 * max(1.0, np.abs(ref).max()), (what, np.abs(got - ref).max())

    for f in range(2):
        od, hd, state = N.forward_D(net, gb[f"k_x{f}"], state)
        close(od.data, gb[f"k_od{f}"], f"od{f}")
        for j, h in enumerate(hd):
            close(h.data, gb[f"k_hd{f}_{j}"], f"hd{f}_{j}")
        fields = N.predict_kernel_fields(net, hd)
        for i, fl in enumerate(fields):
            close(fl.logits.data, gb[f"k_logits{f}_{i}"], f"logits{f}_{i}")
            nz = fl.normalized().data
            close(nz, gb[f"k_norm{f}_{i}"], f"norm{f}_{i}")
            np.testing.assert_allclose(nz.sum(axis=1), 1.0, atol=1e-6)
        img = N.forward_K(net, hd, od)
        close(img.data, gb[f"k_img{f}"], f"img{f}")
    # the split path equals the fused forward_full on the same input and state
    s1 = N.reset_state(net.config, (32, 48))
    o_full, _, _ = N.forward_full(net, gb["k_x0"], s1)
    s2 = N.reset_state(net.config, (32, 48))
    od, hd, _ = N.forward_D(net, gb["k_x0"], s2)
    np.testing.assert_allclose(N.forward_K(net, hd, od).data, o_full.data, rtol=0, atol=1e-6)
    with pytest.raises(ValueError, match="divisible"):
        N.forward_D(net, np.zeros((1, 5, 30, 48), np.float32), N.reset_state(net.config, (30, 48)))


@gpu
@pytest.mark.parametrize("mode", ["full", "naive", "compact", "direct"])
def test_reference_render_flythrough_body_runs_unchanged(mode):
    """The reference's render_flythrough body, unchanged, over the device modules: same frames as
    this package's render_flythrough (the device-resident twin) and the reference's row schema."""
    _torch()
    from reference_callers import render_flythrough as ref_flythrough

    from paper_2209_09965_b200 import renderer as R
    from paper_2209_09965_b200.noise import default_stack
    from paper_2209_09965_b200.sample_maps import FoveaConfig
    from paper_2209_09965_b200.volume import Camera, Light, TransferFunction, make_procedural_volume

    vol = make_procedural_volume("sphere_shells", (32, 32, 32))
    scene = R.Scene(volume=vol, tf=TransferFunction.default(), light=Light(direction=(-1.0, -1.0, -0.5)))
    cams = R.orbit_cameras(R.OrbitPathSpec(n_frames=3), vol, 64, 36)
    fovea = FoveaConfig(focus=(31.5, 17.5), sigma=0.02, base_density=0.1, pixel_scale=0.09)
    kw = dict(mode=mode, noise=default_stack(), fovea=fovea)
    f_ref, rows_ref = ref_flythrough(scene, cams, R.RenderSettings(), rng=np.random.default_rng(3), **kw)
    f_dev, rows_dev = R.render_flythrough(scene, cams, R.RenderSettings(), rng=np.random.default_rng(3), **kw)
    assert len(rows_ref) == len(rows_dev) == 3
    for a, b, ra, rb in zip(f_ref, f_dev, rows_ref, rows_dev):
        assert np.array_equal(a.rgba, b.rgba)
        assert ra[0] == rb[0] and len(ra) == len(rb) == 5
        assert rb[2] > 0 and rb[4] >= rb[2]
    with pytest.raises(ValueError, match="unknown flythrough mode"):
        R.render_flythrough(scene, cams, mode="bogus")
