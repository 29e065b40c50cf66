"""One frame stream split across the GPUs of a node (BASELINE config 5).

The march: every rank computes the full sample mask (microseconds) and marches only its share of
the compacted active-ray list -- 32-ray packets dealt round-robin, so each rank gets a statistically
equal mix of foveal and peripheral rays (fixed screen tiles would be unbalanced by the fovea). The
marched rays become 12-byte records (pixel, RGBA fp16 -- the network input is fp16) and ONE
all_gather_into_tensor (NCCL over NVLink) gives every rank every record; StripShardedPipeline sizes
it per frame by the compacted ray count (ray_capacity), not by the pixel count.

The reconstruction (StripShardedPipeline): each rank owns a strip of rows [a, b) of the padded
frame (a multiple of the network divisor) and runs the unchanged W-Net on a WINDOW [a - E, b + E)
clipped to the frame, E >= the network's per-frame reach (81 rows measured for FULL_BLOCKS; the
default halo is the interval bound of network.py's structure rounded up to the divisor, 96). A
window's owned rows are then exactly the full-frame network's rows (each output pixel is computed
independently of the tile it falls in; tests/test_gpu_parity.py checks bit-identity) PROVIDED its
recurrent inputs -- the decoder hidden states and O_d fed back into the next frame -- are exact
over the whole window. They are exact on the owned rows; after every frame each rank sends its
owned boundary bands (E rows: all four hidden levels + O_d, fv_state_band) to its two neighbours
and receives theirs into its window extension (batch_isend_irecv; the band is the only per-frame
network exchange). Cost: the window's extra rows (2E per interior rank) and ~2 bands per frame.
ShardedFramePipeline (the round-1 design: the march sharded, the network replicated) is kept as
the baseline the strip design replaces.

Kernels: fv_shard_rays, fv_pack_records16, fv_scatter_records16, fv_window_input, fv_state_band
(csrc/shard.cu).
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


def ray_capacity(k: int, world: int) -> int:
    """Per-rank record count for a frame of k compacted rays: the most 32-ray packets any rank owns
    (packets are dealt round-robin, packet_owner), times the packet size; >= one packet."""
    n_packets = (max(int(k), 1) + PACKET - 1) // PACKET
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


# ------------------------------------------------------------------ row-strip reconstruction
def default_halo(config) -> int:
    """Window halo in L0 rows: an interval bound of how far (in rows) the W-Net's output, O_d and
    decoder hidden states of one frame reach (convs widen by one row per conv at their level, a
    2x upsample by two rows of the coarser level, the K stage by one row per filter), rounded up
    to the network divisor. FULL_BLOCKS / DESK_BLOCKS: 95 -> 96 (measured reach: 81)."""
    ne, nd = config.n_enc, config.n_dec
    r, skips = 0, []
    for i in range(ne):
        r += 2 * 2 ** i
        skips.append(r)
    cur, hd = r, {}
    for j in range(nd):
        L = ne - j
        if j > 0:
            cur = max(cur + 2 ** (L + 1), skips[L])
        cur += 2 * 2 ** L
        hd[L] = cur
    img = od = hd[0] + 1
    kinds = [k for k, _ in config.block_config]
    levels = list(range(ne)) + [ne - j for j in range(nd)]
    for i, L in enumerate(levels):
        img = max(img, hd[L]) + 2 ** L
        if kinds[i] == "d" and i < len(kinds) - 1:
            img += 2 ** L
    reach = max(img, od, max(hd.values()))
    div = config.divisor
    return -(-reach // div) * div


def strip_geometry(hp: int, world: int, div: int, halo: int) -> list[tuple[int, int, int, int]]:
    """Per rank (a, b, w0, w1): owned rows [a, b) (multiples of div, as equal as possible) and the
    window [w0, w1) = [a - halo, b + halo] clipped to [0, hp)."""
    if hp % div or halo % div:
        raise ValueError(f"padded height {hp} and halo {halo} must be multiples of {div}")
    units = hp // div
    if units < world:
        raise ValueError(f"{hp} rows cannot be split into {world} strips of {div}-row units")
    out, a = [], 0
    for r in range(world):
        b = a + (units // world + (1 if r < units % world else 0)) * div
        out.append((a, b, max(0, a - halo), min(hp, b + halo)))
        a = b
    if world > 1 and halo > min(b - a for a, b, _, _ in out):
        raise ValueError(f"halo {halo} exceeds the smallest strip; use fewer ranks")
    return out


def band_plan(geo, rank: int):
    """Window-local row ranges of rank's exchanges: {"send_up": (r0, r1), "recv_up": ..., "send_dn",
    "recv_dn"} -- up = with rank - 1, dn = with rank + 1; empty at the frame's edges."""
    a, b, w0, w1 = geo[rank]
    plan = {"send_up": (0, 0), "recv_up": (0, 0), "send_dn": (0, 0), "recv_dn": (0, 0)}
    if rank > 0:
        plan["send_up"] = (a - w0, geo[rank - 1][3] - w0)
        plan["recv_up"] = (0, a - w0)
    if rank + 1 < len(geo):
        plan["send_dn"] = (geo[rank + 1][2] - w0, b - w0)
        plan["recv_dn"] = (b - w0, w1 - w0)
    return plan


def exchange_bands(bufs: dict, rank: int, world: int, group=None) -> None:
    """Send/receive the boundary bands with the two neighbours (batch_isend_irecv; NCCL for CUDA
    tensors, gloo for CPU tensors). bufs: "send_up", "recv_up", "send_dn", "recv_dn" tensors."""
    import torch.distributed as dist

    # gloo moves only host tensors point to point: stage device bands through host copies (the
    # functional check of the torchrun paths on one GPU, FV_DIST_BACKEND=gloo)
    staged = dist.get_backend(group) == "gloo" and any(t.is_cuda for t in bufs.values())
    b = {k: (t.cpu() if staged else t) for k, t in bufs.items()}
    ops = []
    if rank > 0:
        ops += [dist.P2POp(dist.isend, b["send_up"], rank - 1, group),
                dist.P2POp(dist.irecv, b["recv_up"], rank - 1, group)]
    if rank + 1 < world:
        ops += [dist.P2POp(dist.isend, b["send_dn"], rank + 1, group),
                dist.P2POp(dist.irecv, b["recv_dn"], rank + 1, group)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if staged:
        for k in ("recv_up", "recv_dn"):
            if bufs[k].numel():
                bufs[k].copy_(b[k])


class StripShardedPipeline:
    """The C5 frame across `world` GPUs: march sharded by packets, reconstruction by row strips.

    This process is `rank`; emulate=True instead holds every rank's window on this one GPU and runs
    them one after another with the band exchange as device copies (tests: no rank waits on another)."""

    def __init__(self, scene: Scene, net, dims: tuple[int, int], noise: NoiseStack,
                 settings: RenderSettings = RenderSettings(), rank: int = 0, world: int = 1, group=None,
                 halo: int | None = None, emulate: bool = False, size_by_rays: bool = True):
        import ctypes as C

        import torch

        from .network import _DevState

        self.pipe = FramePipeline(scene, None, dims, noise, settings)
        self.net = net
        self.rank, self.world, self.group, self.emulate = rank, world, group, emulate
        self.size_by_rays = size_by_rays
        h, w = dims
        self.h, self.w = h, w
        div = net.config.divisor
        self.hp = -(-h // div) * div
        self.halo = default_halo(net.config) if halo is None else halo
        self.geo = strip_geometry(self.hp, world, div, self.halo)
        ctx = self.pipe.ctx
        self.net_h = net.handle(ctx)
        self.ranks = list(range(world)) if emulate else [rank]
        self.states = {r: _DevState(ctx, self.net_h, self.geo[r][3] - self.geo[r][2], w) for r in self.ranks}
        self.img = {r: torch.empty((self.geo[r][3] - self.geo[r][2], w, 3), dtype=torch.float32, device="cuda")
                    for r in self.ranks}
        n = h * w
        self.bits = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        self.cap = record_capacity(n, world)
        self.rec = torch.empty((self.cap, 3), dtype=torch.int32, device="cuda")
        self.gathered = torch.empty((world * self.cap, 3), dtype=torch.int32, device="cuda")
        self.local_idx = torch.empty((n,), dtype=torch.int32, device="cuda")
        self.local_k = torch.zeros((1,), dtype=torch.int32, device="cuda")
        self.fb = torch.zeros((h, w, 4), dtype=torch.float32, device="cuda")
        self.bands = {}
        for r in self.ranks:
            plan = band_plan(self.geo, r)
            bufs = {}
            for key, (r0, r1) in plan.items():
                nb = C.c_int64()
                _lib.check(ctx.lib.fv_state_band(ctx.h, self.states[r].h, 1, r0, r1 - r0, None, C.byref(nb)))
                bufs[key] = torch.empty((max(1, nb.value),), dtype=torch.uint8, device="cuda")
            self.bands[r] = (plan, bufs)

    def mask(self, fovea: FoveaConfig, frame: int) -> None:
        import ctypes as C

        p = self.pipe
        f = fovea.c_struct()
        _lib.check(p.ctx.lib.fv_mask_compact(p.ctx.h, int(frame), self.h, self.w, C.byref(f), None,
                                             _lib.ptr(self.bits), _lib.ptr(p.idx), _lib.ptr(p.k), None))

    def frame_capacity(self) -> int:
        """Records per rank for the current frame, from its compacted ray count k (every rank
        computed the same full mask, so k -- one 4-byte device read after the mask -- is the same
        on every rank, and so is the all-gather size): ray_capacity(k), not the pixel bound.
        At C5 fast (k ~ 2.8 M of 8.3 M pixels) that gathers about a third of the pixel-sized bytes."""
        if not self.size_by_rays:
            return self.cap
        return min(self.cap, ray_capacity(int(self.pipe.k[0].item()), self.world))

    def march_shard(self, cam: Camera, rank: int, cap: int | None = None) -> None:
        """This rank's packets of the compacted list -> fb -> its first `cap` 12-byte records
        (pixel -1 past its rays)."""
        import ctypes as C

        p = self.pipe
        ctx = p.ctx
        n = self.h * self.w
        _lib.check(ctx.lib.fv_shard_rays(ctx.h, _lib.ptr(p.idx), _lib.ptr(p.k), n, rank, self.world,
                                         _lib.ptr(self.local_idx), _lib.ptr(self.local_k)))
        camc = cam.c_struct()
        _lib.check(ctx.lib.fv_render_sparse(ctx.h, p.vol, C.byref(camc), p._light_ref(), C.byref(p._set),
                                            _lib.ptr(self.local_idx), _lib.ptr(self.local_k), n, _lib.ptr(self.fb),
                                            None, None, None))
        _lib.check(ctx.lib.fv_pack_records16(ctx.h, _lib.ptr(self.fb), _lib.ptr(self.local_idx),
                                             _lib.ptr(self.local_k), self.cap if cap is None else cap,
                                             _lib.ptr(self.rec)))

    def reconstruct_window(self, rank: int, n_records: int | None = None) -> None:
        ctx = self.pipe.ctx
        st = self.states[rank]
        w0 = self.geo[rank][2]
        _lib.check(ctx.lib.fv_window_input(ctx.h, st.h, _lib.ptr(self.bits), self.h, self.w, w0))
        _lib.check(ctx.lib.fv_scatter_records16(ctx.h, st.h, _lib.ptr(self.gathered),
                                                int(self.gathered.shape[0] if n_records is None else n_records),
                                                self.w, w0))
        _lib.check(ctx.lib.fv_reconstruct(ctx.h, self.net_h, st.h, 1, _lib.ptr(self.img[rank]), None, None))

    def _band(self, rank: int, key: str, pack: bool) -> None:
        ctx = self.pipe.ctx
        plan, bufs = self.bands[rank]
        r0, r1 = plan[key]
        if r1 > r0:
            _lib.check(ctx.lib.fv_state_band(ctx.h, self.states[rank].h, 1 if pack else 0, r0, r1 - r0,
                                             _lib.ptr(bufs[key]), None))

    def exchange(self) -> None:
        """After a frame: owned boundary bands -> the neighbours' window extensions."""
        if self.emulate:
            for r in self.ranks:
                for key in ("send_up", "send_dn"):
                    self._band(r, key, True)
            for r in self.ranks:
                if r > 0:
                    self.bands[r][1]["recv_up"].copy_(self.bands[r - 1][1]["send_dn"])
                    self._band(r, "recv_up", False)
                if r + 1 < self.world:
                    self.bands[r][1]["recv_dn"].copy_(self.bands[r + 1][1]["send_up"])
                    self._band(r, "recv_dn", False)
            return
        r = self.rank
        for key in ("send_up", "send_dn"):
            self._band(r, key, True)
        if self.world > 1:
            exchange_bands(self.bands[r][1], r, self.world, self.group)
        for key in ("recv_up", "recv_dn"):
            self._band(r, key, False)

    def step(self, cam: Camera, fovea: FoveaConfig, frame: int) -> None:
        """One frame on this rank: mask, its march share, the record all-gather, its window's
        reconstruction, the band exchange."""
        import torch.distributed as dist

        self.mask(fovea, frame)
        cap = self.frame_capacity()
        self.march_shard(cam, self.rank, cap)
        if self.world > 1:
            dist.all_gather_into_tensor(self.gathered[:self.world * cap], self.rec[:cap], group=self.group)
        else:
            self.gathered[:cap].copy_(self.rec[:cap])
        self.reconstruct_window(self.rank, self.world * cap)
        self.exchange()

    def step_emulated(self, cam: Camera, fovea: FoveaConfig, frame: int) -> None:
        """Every rank's share of the frame on this GPU, one rank after another."""
        self.mask(fovea, frame)
        cap = self.frame_capacity()
        for r in range(self.world):
            self.march_shard(cam, r, cap)
            self.gathered[r * cap:(r + 1) * cap].copy_(self.rec[:cap])
        for r in self.ranks:
            self.reconstruct_window(r, self.world * cap)
        self.exchange()

    def owned_rgb(self, rank: int):
        """The rank's owned rows of the frame's image (rows past the film dropped)."""
        a, b, w0, _ = self.geo[rank]
        return self.img[rank][a - w0:min(b, self.h) - w0]

    @property
    def rgb(self):
        """The whole (H, W, 3) image (emulated runs: every rank's owned rows)."""
        import torch

        return torch.cat([self.owned_rgb(r) for r in self.ranks], dim=0)

