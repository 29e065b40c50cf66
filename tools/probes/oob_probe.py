import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import fovray_oracle as O
from paper_2209_09965_b200 import sample_maps as S
from paper_2209_09965_b200.noise import default_stack
from paper_2209_09965_b200.renderer import RenderSettings, Scene, render_sparse_compact
from paper_2209_09965_b200.volume import Camera, Light, TransferFunction, make_procedural_volume, VolumeGrid
for dims in [(40, 36, 32), (128, 128, 128), (256, 256, 256)]:
    base = make_procedural_volume("sphere_shells", dims)
    for scale, off in [(1.0, 0.0), (1.6, -0.2)]:
        data = base.data.astype(np.float32) * np.float32(scale) + np.float32(off)
        vol = VolumeGrid(base.dims, base.spacing, data, (float(data.min()), float(data.max())), _validated=True)
        sc = Scene(volume=vol, tf=TransferFunction.default(), light=Light(direction=(-1.0, -1.0, -0.5)))
        c = np.array(dims) / 2
        cam = Camera(position=tuple(c + np.array([2.2, 1.7, 2.5]) * dims[0]), look_at=tuple(c), fov_y=45.0, width=256, height=192)
        h, w = cam.height, cam.width
        m = S.build_sample_mask(default_stack(), 0, S.build_tau_map(S.FoveaConfig(focus=((w-1)/2,(h-1)/2), sigma=0.2, base_density=0.3, pixel_scale=S.pixel_scale_for_film((h, w))), (h, w)))
        comp = S.compact_mask(m)
        pix = np.flatnonzero(m.bits.reshape(-1))
        ref = render_sparse_compact(sc, cam, comp, RenderSettings(precision="fp64")).rgba.reshape(-1, 4)[pix]
        got = render_sparse_compact(sc, cam, comp, RenderSettings(), want_depth=False).rgba.reshape(-1, 4)[pix]
        gq = render_sparse_compact(sc, cam, comp, RenderSettings()).rgba.reshape(-1, 4)[pix]
        print(dims, scale, 'filtered max', float(np.abs(got-ref).max()), 'psnr', round(O.psnr(got[:, :3], ref[:, :3]), 1),
              '| quads+filtered-shadow max', float(np.abs(gq-ref).max()), 'psnr', round(O.psnr(gq[:, :3], ref[:, :3]), 1), flush=True)
