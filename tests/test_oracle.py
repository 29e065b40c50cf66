"""The CPU oracle is pinned to the reference: fixtures in tests/golden were produced by running
the unmodified reference package (tests/golden/make_golden.py)."""
import hashlib
import json

import numpy as np
import pytest

from oracle import fovray_oracle as O


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def test_stbn_stack_is_the_reference_default(stack_values):
    # SHA-256 of default_stack() float32 LE values
    assert sha(stack_values.astype("<f4").tobytes()) == \
        "25e032671e1102611b5c2c8032037f58d8625c69635df88cde124426f68605d5"


def test_masks_bit_exact_against_reference(golden, stack_values):
    recs = json.loads((golden / "masks.json").read_text())
    small = np.load(golden / "masks_small.npz")
    for r in recs:
        tau = O.tau_map(r["H"], r["W"], r["focus"], r["sigma"], r["pb"], r["pixel_scale"])
        bits = O.sample_mask(stack_values, r["H"], r["W"], r["frame"], tau)
        idx = O.compact(bits).astype(np.int32)
        assert idx.size == r["k"], r["name"]
        assert sha(np.packbits(bits.ravel()).tobytes()) == r["sha_bits"], r["name"]
        assert sha(idx.tobytes()) == r["sha_idx"], r["name"]
        if r["name"] in small.files:
            assert np.array_equal(bits, small[r["name"]])


def test_cmax_fsum_point():
    # reference tests/test_sample_maps.py:134-152 (fsum oracle at 1280x720, rel 1e-12)
    import math
    tau = O.tau_map(720, 1280, (639.5, 359.5), 0.02, 0.03, 1.0 / 32.0)
    s = 1.0 / 32.0
    acc = []
    for v in range(0, 720, 9):
        dy2 = ((v - 359.5) * s) ** 2
        acc.append(math.fsum(math.exp(-0.5 * (((u - 639.5) * s) ** 2 + dy2) * 0.02) * 0.97 + 0.03
                             for u in range(1280)))
    oracle = math.fsum(acc) / (80 * 1280)
    assert tau[::9].mean() == pytest.approx(oracle, rel=1e-12)


def test_focus_pixel_tau_is_one():
    tau = O.tau_map(16, 16, (7.0, 3.0), 0.04, 0.03, 1.0 / 32)
    assert tau[3, 7] == 1.0


def test_procedural_volumes_bit_exact(golden):
    for r in json.loads((golden / "volumes.json").read_text()):
        d, vr = O.procedural_volume(r["kind"], tuple(r["dims"]))
        assert sha(d.tobytes()) == r["sha"], (r["kind"], r["dims"])
        assert list(vr) == r["value_range"]


def _scene32():
    vol, _ = O.procedural_volume("sphere_shells", (32, 32, 32))
    return vol


LIGHT = ("dir", (-1.0, -1.0, -0.5), (1.0, 1.0, 1.0))
CAM = dict(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0, width=64, height=36)


def test_marcher_reproduces_reference_golden_sha(golden):
    # the reference's own golden image (pkg/tests/test_renderer.py:109-114, :276)
    vol = _scene32()
    rgba, _ = O.render_image(vol, (1, 1, 1), O.DEFAULT_LUT, LIGHT, dict(CAM, width=160, height=90))
    assert sha(rgba.tobytes()) == "be47e7e86eaa47b07c7e0395a753a348844857a618006160f2dcdeead4407c0f"
    meta = json.loads((golden / "render_small.json").read_text())
    assert meta["full160_sha"] == sha(rgba.tobytes())


@pytest.mark.parametrize("key,kw,light", [
    ("full64", {}, LIGHT),
    ("bg64", dict(background=(0.1, 0.2, 0.3, 0.5), early_term_alpha=1.1, step_size=0.37), LIGHT),
    ("nolight64", {}, None),
    ("point64", {}, ("point", (40.0, 50.0, -10.0), (0.9, 1.0, 0.8))),
])
def test_marcher_bit_exact(golden, key, kw, light):
    g = np.load(golden / "render_small.npz")
    rgba, depth = O.render_image(_scene32(), (1, 1, 1), O.DEFAULT_LUT, light, CAM, **kw)
    assert np.array_equal(rgba, g[key + "_rgba"])
    assert np.array_equal(depth, g[key + "_depth"])


def test_sparse_and_anisotropic_bit_exact(golden):
    g = np.load(golden / "render_small.npz")
    rgba, depth = O.render_image(_scene32(), (1, 1, 1), O.DEFAULT_LUT, LIGHT, CAM, bits=g["sparse64_bits"])
    assert np.array_equal(rgba, g["sparse64_rgba"]) and np.array_equal(depth, g["sparse64_depth"])
    vv, _ = O.procedural_volume("vortex_field", (33, 17, 9))
    cam = dict(position=(60.0, 50.0, -30.0), look_at=(16.0, 17.0, 2.0), fov_y=50.0, width=48, height=40,
               up=(0.0, 0.0, 1.0))
    rgba, depth = O.render_image(vv, (1.0, 2.0, 0.5), O.DEFAULT_LUT, ("dir", (0.3, -1.0, 0.2), (1, 1, 1)), cam)
    assert np.array_equal(rgba, g["aniso_rgba"]) and np.array_equal(depth, g["aniso_depth"])


def test_orbit_camera_sparse_frames(golden):
    g = np.load(golden / "render_small.npz")
    meta = json.loads((golden / "render_small.json").read_text())
    vol, _ = O.procedural_volume("sphere_shells", (64, 64, 64))
    for i in (0, 137):
        pos, look = O.orbit_camera(i, 500, (64, 64, 64))
        assert np.allclose(pos, meta[f"orbit{i}_cam"]["position"], rtol=0, atol=0)
        rgba, depth = O.render_image(vol, (1, 1, 1), O.DEFAULT_LUT, LIGHT,
                                     dict(position=pos, look_at=look, fov_y=45.0, width=96, height=96),
                                     bits=g[f"orbit{i}_bits"])
        assert np.array_equal(rgba, g[f"orbit{i}_rgba"])


@pytest.mark.parametrize("tag,blocks,seed,frames,fp16", [
    ("desk", O.DESK_BLOCKS, 7, 2, False), ("deskpad", O.DESK_BLOCKS, 7, 2, False),
    ("full", O.FULL_BLOCKS, 0, 3, True), ("fullwide", O.FULL_BLOCKS, 3, 2, True)])
def test_network_forward_matches_reference(golden, tag, blocks, seed, frames, fp16):
    g = np.load(golden / "net_small.npz")
    p = O.init_params(blocks, seed, fp16_weights=fp16)
    st = None
    for f in range(frames):
        o, od, st = O.net_forward(p, blocks, g[f"{tag}_x{f}"][0], st)
        # fp32 with a different summation order than the reference's BLAS
        np.testing.assert_allclose(o, g[f"{tag}_o{f}"][0], atol=2e-5)
        np.testing.assert_allclose(od, g[f"{tag}_od{f}"][0], atol=2e-5)
    for j, h in enumerate(st["hidden"]):
        np.testing.assert_allclose(h, g[f"{tag}_hidden{j}"][0], atol=2e-5)


def test_psnr_ssim_identity():
    a = np.random.default_rng(0).random((32, 32, 3))
    assert O.psnr(a, a) == 100.0
    assert O.ssim(a, a) == pytest.approx(1.0)


# ---------------------------------------------------------------- compression sweep pieces
def test_uniform_noise_and_direct_draws_match_reference(golden):
    g = np.load(golden / "sweep_small.npz")
    assert np.array_equal(O.uniform_noise(12, 16, 2, seed=5), g["uniform_12x16_s5"])
    tau = O.tau_map(24, 40, (20.0, 11.0), 0.06, 0.07, 0.125)
    assert np.array_equal(O.direct_samples(tau, 400, np.random.default_rng(11)), g["direct_pos"])


def test_naive_and_direct_renders_match_reference(golden):
    g = np.load(golden / "sweep_small.npz")
    for key in ("naive2", "naive20"):
        bits = g[key + "_bits"]
        rgba, depth = O.render_image(_scene32(), (1, 1, 1), O.DEFAULT_LUT, LIGHT, CAM, bits=bits)
        assert np.array_equal(rgba, g[key + "_rgba"]) and np.array_equal(depth, g[key + "_depth"])
        assert O.naive_lanes(bits).size == int(g[key + "_work"])
    pos = g["direct64_pos"]
    flat = np.unique(pos[:, 1] * CAM["width"] + pos[:, 0])
    bits = np.zeros(CAM["height"] * CAM["width"], bool)
    bits[flat] = True
    rgba, depth = O.render_image(_scene32(), (1, 1, 1), O.DEFAULT_LUT, LIGHT, CAM,
                                 bits=bits.reshape(CAM["height"], CAM["width"]))
    assert np.array_equal(rgba, g["direct64_rgba"]) and np.array_equal(depth, g["direct64_depth"])


def test_cmax_settings_rows_match_reference(golden, stack_values):
    g = np.load(golden / "sweep_small.npz")
    h, w = 90, 160
    for pb, sigma, cm, dens in g["cmax_rows"]:
        tau = O.tau_map(h, w, ((w - 1) / 2.0, (h - 1) / 2.0), sigma, pb, 1.0 / 32.0)
        d = np.mean([O.sample_mask(stack_values, h, w, f, tau).mean() for f in range(stack_values.shape[0])])
        assert d == dens
        assert abs(float(np.mean(tau)) - cm) <= 1e-12


# ---------------------------------------------------------------- quality metrics
def test_metric_restatements_match_reference(golden):
    from conftest import metrics_inputs

    g = np.load(golden / "metrics_small.npz")
    a, b, big_a, big_b, seq_p, seq_g = metrics_inputs()
    got = [O.psnr(a, b), O.ssim(a, b), O.msssim(a, b), O.psnr(big_a, big_b), O.ssim(big_a, big_b),
           O.msssim(big_a, big_b), O.psnr(a, a), O.ssim(a, a), O.msssim(a, 1.0 - a),
           O.ssim(np.stack([a[..., 0]] * 3, -1), np.stack([b[..., 0]] * 3, -1)), O.psnr(a, b, peak=2.0)]
    np.testing.assert_allclose(got, g["values"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(O.tpsnr(seq_p, seq_g), g["rep"][3, 1:], rtol=1e-12)
