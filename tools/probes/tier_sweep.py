"""Fast-tier sweep of the frame loop's march (no depth output: filtered main + shadow samples on
volumes >= 128 per axis, else quads + filtered shadow) against the fp64 tier (pinned <= 1e-9 to the
reference): every procedural kind, two sizes, three cameras, two lights; max |err| and PSNR over the
active pixels of a foveated frame."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
from oracle import fovray_oracle as O
from paper_2209_09965_b200 import sample_maps as S
from paper_2209_09965_b200.noise import default_stack
from paper_2209_09965_b200.renderer import RenderSettings, Scene, render_sparse_compact
from paper_2209_09965_b200.volume import Camera, Light, TransferFunction, make_procedural_volume

stack = default_stack()
worst = (0.0, 1e9)
KINDS = sys.argv[1].split(",") if len(sys.argv) > 1 else ["sphere_shells", "vortex_field", "box_lattice"]
for kind in KINDS:
    for n in (64, 128, 256):
        vol = make_procedural_volume(kind, (n, n, n))
        for li, ld in enumerate([(-1.0, -1.0, -0.5), (0.4, -1.0, 0.7)]):
            sc = Scene(volume=vol, tf=TransferFunction.default(), light=Light(direction=ld))
            for ci, (dx, dy, dz) in enumerate([(2.2, 1.7, 2.5), (-2.6, 0.9, 1.4), (0.6, 2.8, -1.9)]):
                c = np.array([n / 2.0] * 3)
                cam = Camera(position=tuple(c + np.array([dx, dy, dz]) * n), look_at=tuple(c), fov_y=40.0,
                             width=320, height=240)
                h, w = cam.height, cam.width
                m = S.build_sample_mask(stack, ci, S.build_tau_map(S.FoveaConfig(
                    focus=((w - 1) / 2, (h - 1) / 2), sigma=0.06, base_density=0.07,
                    pixel_scale=S.pixel_scale_for_film((h, w))), (h, w)))
                comp = S.compact_mask(m)
                pix = np.flatnonzero(m.bits.reshape(-1))
                ref = render_sparse_compact(sc, cam, comp, RenderSettings(precision="fp64")).rgba.reshape(-1, 4)[pix]
                got = render_sparse_compact(sc, cam, comp, RenderSettings(), want_depth=False).rgba.reshape(-1, 4)[pix]
                mx = float(np.abs(got - ref).max())
                ps = O.psnr(got[:, :3], ref[:, :3])
                worst = (max(worst[0], mx), min(worst[1], ps))
                flag = "" if (mx <= 1e-2 and ps >= 80) else "  <-- outside the fast tier"
                print(f"{kind:14s} {n:4d} light{li} cam{ci}: max {mx:.2e} psnr {ps:6.1f}{flag}", flush=True)
print(f"worst: max {worst[0]:.2e}, psnr {worst[1]:.1f}")
