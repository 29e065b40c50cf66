"""One frame stream split across the GPUs of a node (BASELINE config 5).

Every rank computes the full sample mask (microseconds) and marches only its share of the
compacted active-ray list: 32-ray packets dealt round-robin, so each rank gets a statistically
equal mix of foveal and peripheral rays (fixed screen tiles would be unbalanced by the fovea). The
marched (pixel, RGBA) records of all ranks are all-gathered -- NCCL over NVLink on the GPU box --
and scattered into the network input exactly as the marcher writes it, so every rank reconstructs
the same frame as the unsharded pipeline (bit-exact; tests/test_gpu_parity.py emulates the ranks
on one GPU, tests/test_multi.py runs the exchange with gloo). The recurrent network needs the whole
frame, so reconstruction is replicated; marching -- which dominates at 1024^3 -- scales.

Kernels: fv_shard_rays, fv_pack_records, fv_scatter_records (csrc/shard.cu).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .noise import NoiseStack
from .pipeline import FramePipeline
from .renderer import RenderSettings, Scene
from .sample_maps import FoveaConfig
from .volume import Camera

PACKET = 32


def packet_owner(k: int, world: int) -> np.ndarray:
    """Rank owning each of the k compacted rays (host mirror of shard_rays_kernel)."""
    return (np.arange(k) // PACKET) % world


def record_capacity(n_pixels: int, world: int) -> int:
    """Fixed per-rank record count: the most packets any rank can own, times the packet size."""
    n_packets = (n_pixels + PACKET - 1) // PACKET
    return (n_packets + world - 1) // world * PACKET


def all_gather_records(pix, rgba, world: int, group=None):
    """All-gather fixed-capacity (pixel, RGBA) records over the process group (NCCL for CUDA
    tensors, gloo for CPU tensors); returns the concatenated (world*cap,) and (world*cap, 4)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return pix, rgba
    gp = [torch.empty_like(pix) for _ in range(world)]
    gr = [torch.empty_like(rgba) for _ in range(world)]
    dist.all_gather(gp, pix, group=group)
    dist.all_gather(gr, rgba, group=group)
    return torch.cat(gp), torch.cat(gr)


def scatter_records_host(pix: np.ndarray, rgba: np.ndarray, h: int, w: int) -> np.ndarray:
    """Host mirror of scatter_records_kernel into an (H, W, 4) frame (records with pixel < 0 skipped)."""
    out = np.zeros((h * w, 4), np.float32)
    sel = pix >= 0
    out[pix[sel]] = rgba[sel]
    return out.reshape(h, w, 4)


class ShardedFramePipeline:
    """FramePipeline whose march is split across `world` ranks (this process is `rank`)."""

    def __init__(self, scene: Scene, net, dims: tuple[int, int], noise: NoiseStack,
                 settings: RenderSettings = RenderSettings(), rank: int = 0, world: int = 1, group=None):
        import torch

        self.pipe = FramePipeline(scene, net, dims, noise, settings)
        self.rank, self.world, self.group = rank, world, group
        h, w = dims
        n = h * w
        self.cap = record_capacity(n, world)
        self.local_idx = torch.empty((n,), dtype=torch.int32, device="cuda")
        self.local_k = torch.zeros((1,), dtype=torch.int32, device="cuda")
        self.fb = torch.zeros((h, w, 4), dtype=torch.float32, device="cuda")
        self.rec_pix = torch.empty((self.cap,), dtype=torch.int32, device="cuda")
        self.rec_rgba = torch.empty((self.cap, 4), dtype=torch.float32, device="cuda")

    @property
    def rgb(self):
        return self.pipe.rgb

    def render_shard(self, cam: Camera, fovea: FoveaConfig, frame: int, rank: int | None = None,
                     mask: bool = True):
        """Mask (all pixels) + this rank's share of the march -> its (pixel, RGBA) records."""
        import ctypes as C

        p = self.pipe
        ctx = p.ctx
        rank = self.rank if rank is None else rank
        if mask:
            p.mask(fovea, frame)  # writes net-input channels 0..4 (zeros + mask) and the compacted list
        n = p.h * p.w
        _lib.check(ctx.lib.fv_shard_rays(ctx.h, _lib.ptr(p.idx), _lib.ptr(p.k), n, rank, self.world,
                                         _lib.ptr(self.local_idx), _lib.ptr(self.local_k)))
        camc = cam.c_struct()
        _lib.check(ctx.lib.fv_render_sparse(ctx.h, p.vol, C.byref(camc), p._light_ref(), C.byref(p._set),
                                            _lib.ptr(self.local_idx), _lib.ptr(self.local_k), n, _lib.ptr(self.fb),
                                            None, None, None))
        _lib.check(ctx.lib.fv_pack_records(ctx.h, _lib.ptr(self.fb), _lib.ptr(self.local_idx),
                                           _lib.ptr(self.local_k), self.cap, _lib.ptr(self.rec_pix),
                                           _lib.ptr(self.rec_rgba)))
        return self.rec_pix, self.rec_rgba

    def finish(self, pix, rgba) -> None:
        """Scatter the gathered records into the network input and reconstruct."""
        p = self.pipe
        ctx = p.ctx
        _lib.check(ctx.lib.fv_scatter_records(ctx.h, p.state.h, _lib.ptr(pix), _lib.ptr(rgba), int(pix.numel()),
                                              p.w, None))
        p.reconstruct()

    def step(self, cam: Camera, fovea: FoveaConfig, frame: int) -> None:
        pix, rgba = self.render_shard(cam, fovea, frame)
        gp, gr = all_gather_records(pix, rgba, self.world, self.group)  # stream-ordered after the pack
        self.finish(gp, gr)

    def step_emulated(self, cam: Camera, fovea: FoveaConfig, frame: int) -> None:
        """All `world` ranks' shares on this one GPU, one after another (tests; no rank waits on
        another), then the same scatter + reconstruction."""
        import torch

        pixs, rgbas = [], []
        for r in range(self.world):
            pix, rgba = self.render_shard(cam, fovea, frame, rank=r, mask=(r == 0))
            pixs.append(pix.clone())
            rgbas.append(rgba.clone())
        self.finish(torch.cat(pixs), torch.cat(rgbas))
