"""Generate the committed golden fixtures by running the REFERENCE package.

Run in the dev container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Every fixture written here is produced by the unmodified reference
(`/root/reference/pkg/src/fovray`) through its public functions; nothing
from this repository is imported. The fixtures pin the oracle (`oracle/`)
in the CPU test-suite and are the targets of the GPU parity tests.

Outputs (all under tests/golden/ unless noted):
  paper_2209_09965_b200/data/stbn_64x64x8_s1.noise  default_stack() in RNKSTACK form
  masks.json            frame-mask k + SHA-256 of packbits(bits) and of int32 v*W+u
  masks_small.npz       full bit arrays for small films
  volumes.json/.npz     make_procedural_volume hashes + small arrays
  render_small.npz      render_full / render_sparse_compact outputs on small scenes
  net_small.npz         forward_full outputs (desk + paper nets, carried state)
  e2e_c1.npz            config C1 (64^3, 256x256, fast) mask -> march -> fp16 net, 2 frames
  rawvol_small.npz      load_raw_volume on uint8 / float32 / constant / NaN raw files
  viewer_small.npz      viewer.RenderService.render_frame: decoded PNGs + headers, every mode
  metrics_small.npz     PSNR / SSIM / MS-SSIM / tPSNR / quality-report values on seeded images
  sweep_small.npz       compression sweep pieces: uniform noise, direct draws, naive/direct
                        renders, foveated-settings density rows
  boundary_small.npz    generate_rays, sample_trilinear, TransferFunction.apply, tile_field /
                        tile_lookup, foveal_density, forward_D / predict_kernel_fields / forward_K
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from fovray import noise as rn  # noqa: E402
from fovray import sample_maps as rsm  # noqa: E402
from fovray import renderer as rr  # noqa: E402
from fovray import volume as rv  # noqa: E402
from fovray import network as rnet  # noqa: E402
from fovray import bench as rb  # noqa: E402
from fovray.autograd import no_grad  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
DATA = REPO / "paper_2209_09965_b200" / "data"


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def mask_record(stack, name, h, w, frame, focus, sigma, pb, scale):
    cfg = rsm.FoveaConfig(focus=focus, sigma=sigma, base_density=pb, pixel_scale=scale)
    tau = rsm.build_tau_map(cfg, (h, w))
    m = rsm.build_sample_mask(stack, frame, tau)
    comp = rsm.compact_mask(m)
    flat = (comp.coords[:, 1] * w + comp.coords[:, 0]).astype(np.int32)
    margin = float(np.min(np.abs(tau.values - rn.tile_field(stack, h, w, frame).astype(np.float64))))
    return {
        "name": name, "H": h, "W": w, "frame": frame, "focus": list(map(float, focus)),
        "sigma": sigma, "pb": pb, "pixel_scale": scale, "k": int(comp.count),
        "sha_bits": sha(np.packbits(m.bits.ravel()).tobytes()),
        "sha_idx": sha(flat.tobytes()), "c_max": rsm.c_max(tau), "min_margin": margin,
    }, m.bits


def gen_masks(stack):
    recs = []
    small = {}
    presets = {"fast": rsm.FAST_PRESET, "hifi": rsm.HIFI_PRESET}
    for (h, w) in [(256, 256), (1080, 1920), (2160, 3840)]:
        scale = rsm.pixel_scale_for_film((h, w))
        for mode, p in presets.items():
            frames = [0, 1, 2, 3] if (h, w) == (1080, 1920) else [0]
            for f in frames:
                r, _ = mask_record(stack, f"{w}x{h}_{mode}_f{f}", h, w, f,
                                   ((w - 1) / 2.0, (h - 1) / 2.0), p["sigma"],
                                   p["base_density"], scale)
                recs.append(r)
    # config-4 moving gaze: fx=(W-1)/2+0.4W sin(2 pi i/500), fy=(H-1)/2+0.4H sin(4 pi i/500)
    h, w = 1080, 1920
    scale = rsm.pixel_scale_for_film((h, w))
    for i in [0, 37, 125, 250, 333, 499]:
        fx = (w - 1) / 2.0 + 0.4 * w * np.sin(2 * np.pi * i / 500)
        fy = (h - 1) / 2.0 + 0.4 * h * np.sin(4 * np.pi * i / 500)
        r, _ = mask_record(stack, f"gaze_hifi_i{i}", h, w, i, (fx, fy),
                           rsm.HIFI_PRESET["sigma"], rsm.HIFI_PRESET["base_density"], scale)
        recs.append(r)
    # small films, random configs, full bit arrays kept
    rng = np.random.default_rng(1234)
    for j, (h, w) in enumerate([(36, 64), (90, 160), (1, 7), (17, 5), (100, 129)]):
        focus = (float(rng.uniform(-10, w + 10)), float(rng.uniform(-10, h + 10)))
        sigma = float(rng.uniform(0.0, 2.0))
        pb = float(rng.uniform(0.0, 1.0))
        scale = float(rng.uniform(0.01, 0.5))
        r, bits = mask_record(stack, f"small{j}", h, w, j * 3, focus, sigma, pb, scale)
        recs.append(r)
        small[f"small{j}"] = bits
    # edge: tau identically 1 (sigma 0) and base density 0
    r, bits = mask_record(stack, "all_on", 40, 70, 5, (3.0, 4.0), 0.0, 0.0, 1.0 / 32)
    recs.append(r)
    small["all_on"] = bits
    r, bits = mask_record(stack, "focus_only", 40, 70, 6, (30.0, 20.0), 1e9, 0.0, 1.0)
    recs.append(r)
    small["focus_only"] = bits
    (HERE / "masks.json").write_text(json.dumps(recs, indent=1))
    np.savez_compressed(HERE / "masks_small.npz", **small)
    print(f"masks: {len(recs)} records")


def gen_volumes():
    recs = []
    arrs = {}
    for kind in ("sphere_shells", "vortex_field", "box_lattice"):
        for dims in [(8, 8, 8), (16, 12, 10), (32, 32, 32), (64, 64, 64), (33, 17, 9)]:
            v = rv.make_procedural_volume(kind, dims)
            recs.append({"kind": kind, "dims": list(dims), "sha": sha(v.data.tobytes()),
                         "value_range": list(map(float, v.value_range))})
            if dims in [(16, 12, 10), (33, 17, 9)]:
                arrs[f"{kind}_{dims[0]}x{dims[1]}x{dims[2]}"] = v.data
    (HERE / "volumes.json").write_text(json.dumps(recs, indent=1))
    np.savez_compressed(HERE / "volumes.npz", **arrs)
    print("volumes done")


def test_scene():
    vol = rv.make_procedural_volume("sphere_shells", (32, 32, 32))
    return rr.Scene(volume=vol, tf=rv.TransferFunction.default(),
                    light=rv.Light(direction=(-1.0, -1.0, -0.5), intensity=(1.0, 1.0, 1.0)))


def gen_renders(stack):
    out = {}
    meta = {}
    scene = test_scene()
    cam = rv.Camera(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0,
                    width=64, height=36)
    fr = rr.render_full(scene, cam)
    out["full64_rgba"], out["full64_depth"] = fr.rgba, fr.depth
    cam160 = rv.Camera(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0,
                       width=160, height=90)
    fr = rr.render_full(scene, cam160)
    out["full160_rgba"], out["full160_depth"] = fr.rgba, fr.depth
    meta["full160_sha"] = sha(fr.rgba.tobytes())
    # sparse compact on a foveated mask of the default stack
    cfg = rsm.FoveaConfig(focus=(40.0, 12.0), sigma=0.3, base_density=0.15, pixel_scale=0.2)
    mask = rsm.build_sample_mask(stack, 3, rsm.build_tau_map(cfg, (36, 64)))
    sp = rr.render_sparse_compact(scene, cam, rsm.compact_mask(mask))
    out["sparse64_rgba"], out["sparse64_depth"], out["sparse64_bits"] = sp.rgba, sp.depth, mask.bits
    # settings variants: background, no early termination, explicit step
    st = rr.RenderSettings(background=(0.1, 0.2, 0.3, 0.5), early_term_alpha=1.1, step_size=0.37)
    fr = rr.render_full(scene, cam, st)
    out["bg64_rgba"], out["bg64_depth"] = fr.rgba, fr.depth
    # no light
    nl = rr.Scene(volume=scene.volume, tf=scene.tf, light=None)
    fr = rr.render_full(nl, cam)
    out["nolight64_rgba"], out["nolight64_depth"] = fr.rgba, fr.depth
    # point light
    pl = rr.Scene(volume=scene.volume, tf=scene.tf,
                  light=rv.Light(position=(40.0, 50.0, -10.0), intensity=(0.9, 1.0, 0.8)))
    fr = rr.render_full(pl, cam)
    out["point64_rgba"], out["point64_depth"] = fr.rgba, fr.depth
    # anisotropic volume: vortex 33x17x9, spacing (1, 2, 0.5)
    vv = rv.make_procedural_volume("vortex_field", (33, 17, 9), spacing=(1.0, 2.0, 0.5))
    sv = rr.Scene(volume=vv, tf=rv.TransferFunction.default(),
                  light=rv.Light(direction=(0.3, -1.0, 0.2)))
    c2 = rv.Camera(position=(60.0, 50.0, -30.0), look_at=(16.0, 17.0, 2.0), fov_y=50.0,
                   width=48, height=40, up=(0.0, 0.0, 1.0))
    fr = rr.render_full(sv, c2)
    out["aniso_rgba"], out["aniso_depth"] = fr.rgba, fr.depth
    # C1 scene, orbit frame 0 of a 500-frame path, 96x96, hifi mask
    vol64 = rv.make_procedural_volume("sphere_shells", (64, 64, 64))
    s64 = rr.Scene(volume=vol64, tf=rv.TransferFunction.default(),
                   light=rv.Light(direction=(-1.0, -1.0, -0.5), intensity=(1.0, 1.0, 1.0)))
    cams = rr.orbit_cameras(rr.OrbitPathSpec(n_frames=500), vol64, 96, 96)
    for i in (0, 137):
        c = cams[i]
        cfg = rsm.FoveaConfig(focus=(47.5, 47.5), sigma=0.06, base_density=0.07,
                              pixel_scale=rsm.pixel_scale_for_film((96, 96)))
        mask = rsm.build_sample_mask(stack, i, rsm.build_tau_map(cfg, (96, 96)))
        sp = rr.render_sparse_compact(s64, c, rsm.compact_mask(mask))
        out[f"orbit{i}_rgba"], out[f"orbit{i}_depth"], out[f"orbit{i}_bits"] = sp.rgba, sp.depth, mask.bits
        meta[f"orbit{i}_cam"] = {"position": list(c.position), "look_at": list(c.look_at)}
    np.savez_compressed(HERE / "render_small.npz", **out)
    (HERE / "render_small.json").write_text(json.dumps(meta, indent=1))
    print("renders done")


def gen_sweep(stack):
    """Compression-sweep inputs and outputs: uniform noise, direct draws, naive/direct renders,
    foveated-settings density rows (bench.cmd_bench_cmax's building blocks)."""
    out = {}
    un = rn.gen_uniform_noise(12, 16, 2, seed=5)
    out["uniform_12x16_s5"] = un.values
    cfg = rsm.FoveaConfig(focus=(20.0, 11.0), sigma=0.06, base_density=0.07, pixel_scale=0.125)
    out["direct_pos"] = rsm.draw_direct_samples(cfg, np.zeros((24, 40)), 400, np.random.default_rng(11))
    scene = test_scene()
    cam = rv.Camera(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0,
                    width=64, height=36)
    un2 = rn.gen_uniform_noise(36, 64, 1, seed=2)
    for tau in (0.02, 0.2):
        mask = rsm.build_sample_mask(un2, 0, rsm.TauMap(values=np.full((36, 64), tau)))
        nv = rr.render_sparse_naive(scene, cam, mask)
        key = f"naive{int(tau * 100)}"
        out[key + "_rgba"], out[key + "_depth"], out[key + "_bits"] = nv.rgba, nv.depth, mask.bits
        out[key + "_work"] = np.array(nv.work_items)
    pos = rsm.draw_direct_samples(rsm.FoveaConfig(focus=(32.0, 18.0), sigma=0.3, base_density=0.1,
                                                  pixel_scale=0.2), np.zeros((36, 64)), 300,
                                  np.random.default_rng(3))
    dr = rr.render_sparse_direct(scene, cam, pos)
    out["direct64_pos"], out["direct64_rgba"], out["direct64_depth"] = pos, dr.rgba, dr.depth
    rows = rsm.cmax_sweep_rows([(0.03, 0.02), (0.07, 0.06), (0.01, 0.02), (0.10, 0.02)], stack, (90, 160))
    out["cmax_rows"] = np.array(rows, dtype=np.float64)
    np.savez_compressed(HERE / "sweep_small.npz", **out)
    print("sweep done")


def metrics_inputs():
    """Seeded inputs of the metric fixtures (rebuilt identically by the tests: PCG64 streams)."""
    rng = np.random.default_rng(21)
    a = rng.random((64, 80, 3))
    b = np.clip(a + 0.05 * rng.standard_normal(a.shape), 0, 1)
    yy, xx = np.mgrid[0:192, 0:256]
    big_a = np.stack([np.exp(-((xx - 90 - 20 * c) ** 2 + (yy - 100) ** 2) / 3000.0) for c in range(3)], -1)
    big_b = np.clip(big_a + 0.02 * rng.standard_normal(big_a.shape), 0, 1)
    s = a[:32, :40]
    seq_p = [np.clip(s + 0.03 * k + 0.02 * rng.standard_normal(s.shape), 0, 1) for k in range(4)]
    seq_g = [np.clip(s + 0.03 * k, 0, 1) for k in range(4)]
    return a, b, big_a, big_b, seq_p, seq_g


def gen_metrics():
    """metrics.psnr / ssim / msssim / tpsnr / build_quality_report on seeded images."""
    from fovray import metrics as rm

    a, b, big_a, big_b, seq_p, seq_g = metrics_inputs()
    vals = [rm.psnr(a, b), rm.ssim(a, b), rm.msssim(a, b), rm.psnr(big_a, big_b), rm.ssim(big_a, big_b),
            rm.msssim(big_a, big_b), rm.psnr(a, a), rm.ssim(a, a), rm.msssim(a, 1.0 - a),
            rm.ssim(a[..., 0], b[..., 0]), rm.psnr(a, b, peak=2.0)]
    rep = rm.build_quality_report(seq_p, seq_g)
    np.savez_compressed(HERE / "metrics_small.npz", values=np.array(vals),
                        rep=np.stack([rep.psnr, rep.ssim, rep.msssim, rep.tpsnr]))
    print("metrics done")


def gen_viewer(stack):
    """viewer.RenderService.render_frame messages (decoded PNGs + headers) for every mode."""
    import io as _io

    from PIL import Image
    from fovray import bench as rbench
    from fovray import viewer as rview

    scene = test_scene()
    net = rbench._quantized_net(rnet.init_network(rnet.NetConfig.from_string(rnet.DESK_BLOCKS), seed=7), "fp16")
    cam = rv.Camera(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0, width=64, height=36)
    svc = rview.RenderService(scene, film=(64, 36), checkpoint=net, noise=stack,
                              settings=rr.RenderSettings(step_size=1.0), camera=cam)
    out = {}
    state = rview.default_session((64, 36))
    plan = [("sparse_raw", {}), ("reconstructed", {}), ("reconstructed", {"focus": [10.0, 30.0], "p_b": 0.2}),
            ("ground_truth", {}), ("side_by_side", {"sigma": 0.5})]
    for i, (mode, ctl) in enumerate(plan):
        msg = dict(ctl, mode=mode)
        state = rview.handle_control(state, msg, svc.film, has_checkpoint=True)
        blob, state = svc.render_frame(state)
        d = rview.parse_frame_message(blob)
        out[f"img{i}"] = np.asarray(Image.open(_io.BytesIO(d["png"])))
        out[f"hdr{i}"] = np.array([d["frame_id"], d["width"], d["height"], rview.MODES.index(d["mode"]),
                                   d["focus"][0], d["focus"][1], d["p_b"], d["sigma"]], dtype=np.float64)
    np.savez_compressed(HERE / "viewer_small.npz", **out)
    print("viewer done")


def gen_rawvol():
    """volume.load_raw_volume on small raw files (uint8, float32, constant, NaN)."""
    import tempfile

    rng = np.random.default_rng(9)
    out = {}
    cases = {"u8": (rng.integers(0, 256, size=(9, 10, 12), dtype=np.uint8), "uint8"),
             "f32": ((rng.standard_normal((9, 10, 12)) * 3.7 + 1.1).astype("<f4"), "float32"),
             "const": (np.full((9, 10, 12), 2.5, dtype="<f4"), "float32")}
    with tempfile.TemporaryDirectory() as d:
        for key, (arr, dt) in cases.items():
            path = Path(d) / f"{key}.raw"
            path.write_bytes(arr.tobytes())
            vg = rv.load_raw_volume(path, rv.VolumeMeta(dims=(12, 10, 9), dtype=dt, spacing=(1.0, 2.0, 0.5)))
            out[key + "_raw"] = arr
            out[key + "_data"] = vg.data
            out[key + "_range"] = np.array(vg.value_range)
        bad = cases["f32"][0].copy()
        bad.reshape(-1)[437] = np.nan
        path = Path(d) / "nan.raw"
        path.write_bytes(bad.tobytes())
        try:
            rv.load_raw_volume(path, rv.VolumeMeta(dims=(12, 10, 9), dtype="float32"))
        except ValueError as e:
            out["nan_msg"] = np.array(str(e))
        out["nan_raw"] = bad
    np.savez_compressed(HERE / "rawvol_small.npz", **out)
    print("rawvol done")


def gen_net():
    out = {}
    rng = np.random.default_rng(77)

    def rand_input(h, w):
        rgba = rng.random((1, 4, h, w)).astype(np.float32)
        m = (rng.random((1, 1, h, w)) < 0.25).astype(np.float32)
        return np.concatenate([rgba * m, m], axis=1)

    cases = [("desk", rnet.DESK_BLOCKS, 7, 32, 32, 2), ("deskpad", rnet.DESK_BLOCKS, 7, 50, 70, 2),
             ("full", rnet.FULL_BLOCKS, 0, 64, 64, 3), ("fullwide", rnet.FULL_BLOCKS, 3, 24, 136, 2)]
    for tag, blocks, seed, h, w, frames in cases:
        net = rnet.init_network(rnet.NetConfig.from_string(blocks), seed=seed)
        if tag.startswith("full"):
            net = rb._quantized_net(net, "fp16")
        state = rnet.reset_state(net.config, (h, w))
        for f in range(frames):
            x = rand_input(h, w)
            with no_grad():
                o, od, state = rnet.forward_full(net, x, state)
            out[f"{tag}_x{f}"] = x
            out[f"{tag}_o{f}"] = o.data
            out[f"{tag}_od{f}"] = od.data
        for j, hd in enumerate(state.hidden):
            out[f"{tag}_hidden{j}"] = hd.data
        with no_grad():
            o2, od2, _ = rnet.forward_full(net, rand_input(h, w), rnet.reset_state(net.config, (h, w)),
                                           use_kernel_stage=False)
        out[f"{tag}_direct_o"] = o2.data
    np.savez_compressed(HERE / "net_small.npz", **out)
    print("net done")


def gen_c1(stack):
    """C1: 64^3 sphere_shells, 256x256, fast, FULL_BLOCKS seed 0 fp16, 2 carried frames."""
    h = w = 256
    scene = rb.default_scene("sphere_shells", (64, 64, 64))
    cams = rr.orbit_cameras(rr.OrbitPathSpec(n_frames=500), scene.volume, w, h)
    spec = rb.ExperimentSpec(dataset="sphere_shells", mode="fast", width=w, height=h)
    fovea = spec.fovea()
    net = rb._quantized_net(rnet.init_network(rnet.NetConfig.from_string(rnet.FULL_BLOCKS), seed=0), "fp16")
    state = rnet.reset_state(net.config, (h, w))
    out = {}
    for i in range(2):
        t0 = time.perf_counter()
        tau = rsm.build_tau_map(fovea, (h, w))
        mask = rsm.build_sample_mask(stack, i, tau)
        comp = rsm.compact_mask(mask)
        fr = rr.render_sparse_compact(scene, cams[i], comp)
        img, state = rb._reconstruct_frame(net, fr.rgba, mask.bits, state)
        out[f"bits{i}"] = mask.bits
        out[f"rgba{i}"] = fr.rgba
        out[f"depth{i}"] = fr.depth
        out[f"img{i}"] = img.astype(np.float32)
        print(f"c1 frame {i}: k={comp.count} {time.perf_counter() - t0:.1f}s")
    np.savez_compressed(HERE / "e2e_c1.npz", **out)


def gen_boundary(stack):
    """The per-sample building blocks and the kernel-stage API of the reference, for the device
    boundary functions: generate_rays, sample_trilinear, TransferFunction.apply, tile_field,
    foveal_density, forward_D / predict_kernel_fields / forward_K."""
    from fovray import autograd as ag

    out = {}
    cam = rv.Camera(position=(80.0, 60.0, 90.0), look_at=(16.0, 16.0, 16.0), fov_y=40.0, width=64, height=36)
    rng = np.random.default_rng(31)
    us = rng.integers(0, 64, 200)
    vs = rng.integers(0, 36, 200)
    o, d = rv.generate_rays(cam, us, vs)
    out.update(ray_us=us, ray_vs=vs, ray_o=o, ray_d=d)
    vol = rv.make_procedural_volume("vortex_field", (33, 17, 9), spacing=(1.0, 2.0, 0.5))
    pts = np.concatenate([rng.uniform(-2, 36, (400, 3)) * np.array([1.0, 1.0, 0.5]),
                          rng.uniform(0, 0.6, (100, 3)), rng.uniform(0, 1, (50, 3)) * vol.extent])
    out.update(tri_pts=pts, tri_vals=rv.sample_trilinear(vol, pts))
    s = np.concatenate([rng.uniform(-0.5, 1.5, 300), [0.0, 1.0, 1.0 / 6, 0.5]])
    out.update(tf_s=s, tf_rgba=rv.TransferFunction.default().apply(s))
    out["tile_field"] = rn.tile_field(stack, 70, 150, 11)
    out["tile_lookup"] = np.array([rn.tile_lookup(stack, u, v, f) for u, v, f in [(0, 0, 0), (70, 3, 9), (-3, 200, 13)]])
    dx = np.arange(-40, 41, dtype=np.float64)[None, :]
    dy = np.arange(-20, 21, dtype=np.float64)[:, None]
    out["fovd"] = rsm.foveal_density((dx, dy), 0.06, 0.02)
    # the kernel stage through the reference's split API, state carried over 2 frames
    net = rnet.init_network(rnet.NetConfig.from_string(rnet.DESK_BLOCKS), seed=5)
    state = rnet.reset_state(net.config, (32, 48))
    for f in range(2):
        x = rng.random((1, 5, 32, 48)).astype(np.float32)
        with no_grad():
            od, hd, state = rnet.forward_D(net, x, state)
            fields = rnet.predict_kernel_fields(net, hd)
            img = rnet.forward_K(net, hd, od)
        out[f"k_x{f}"] = x
        out[f"k_od{f}"] = od.data
        out[f"k_img{f}"] = img.data
        for j, h in enumerate(hd):
            out[f"k_hd{f}_{j}"] = h.data
        for i, fl in enumerate(fields):
            out[f"k_logits{f}_{i}"] = fl.logits.data
            out[f"k_norm{f}_{i}"] = fl.normalized().data
    np.savez_compressed(HERE / "boundary_small.npz", **out)
    print("boundary: done")


def main():
    t0 = time.perf_counter()
    DATA.mkdir(parents=True, exist_ok=True)
    stack = rn.default_stack()
    rn.save_stack(stack, DATA / "stbn_64x64x8_s1.noise")
    print(f"stbn sha {sha(stack.values.astype('<f4').tobytes())}")
    which = set(sys.argv[1:]) or {"masks", "volumes", "renders", "net", "c1", "sweep", "metrics", "viewer", "rawvol",
                                  "boundary"}
    if "masks" in which:
        gen_masks(stack)
    if "volumes" in which:
        gen_volumes()
    if "renders" in which:
        gen_renders(stack)
    if "net" in which:
        gen_net()
    if "c1" in which:
        gen_c1(stack)
    if "sweep" in which:
        gen_sweep(stack)
    if "metrics" in which:
        gen_metrics()
    if "viewer" in which:
        gen_viewer(stack)
    if "rawvol" in which:
        gen_rawvol()
    if "boundary" in which:
        gen_boundary(stack)
    print(f"done in {time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    main()
