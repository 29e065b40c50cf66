"""Device-resident per-frame pipeline: mask -> compaction -> march -> reconstruction.

One FramePipeline owns everything a frame touches on the GPU (volume view, fp16
weights, recurrent state + activations, compacted index list) and launches the
whole of bench.cmd_bench_throughput's loop body (pkg/src/fovray/bench.py:194-209)
without host round trips: the mask kernel writes channels 0..4 of the network
input, the marcher writes the RGBA of active pixels into it, the network reads
it, and the D.head epilogue writes next frame's O_d feedback into channels 5..7.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .network import WNetParams, _DevState
from .noise import NoiseStack
from .renderer import RenderSettings, Scene
from .sample_maps import FoveaConfig
from .volume import Camera


class FramePipeline:
    def __init__(self, scene: Scene, net: WNetParams | None, dims: tuple[int, int], noise: NoiseStack,
                 settings: RenderSettings = RenderSettings(), ctx: _lib.Context | None = None):
        import torch

        self.ctx = ctx or _lib.context()
        self.ctx.ensure_noise(noise)
        self.scene = scene
        self.h, self.w = dims
        self.settings = settings
        self._set = settings.c_struct()
        self._light = scene.light.c_struct() if scene.light is not None else None
        self.vol = scene.volume.handle(self.ctx, scene.tf)
        self.net = net
        self.net_h = net.handle(self.ctx) if net is not None else None
        self.state = _DevState(self.ctx, self.net_h, self.h, self.w) if net is not None else None
        n = self.h * self.w
        self.idx = torch.empty((n,), dtype=torch.int32, device="cuda")
        self.k = torch.zeros((1,), dtype=torch.int32, device="cuda")
        self.rgb = torch.empty((self.h, self.w, 3), dtype=torch.float32, device="cuda")
        self.dense_rgba = None
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def reset(self) -> None:
        if self.state is not None:
            _lib.check(self.ctx.lib.fv_state_reset(self.ctx.h, self.state.h))

    def _light_ref(self):
        return C.byref(self._light) if self._light is not None else None

    def mask(self, fovea: FoveaConfig, frame: int) -> None:
        f = fovea.c_struct()
        _lib.check(self.ctx.lib.fv_mask_compact(self.ctx.h, int(frame), self.h, self.w, C.byref(f), None,
                                                None, _lib.ptr(self.idx), _lib.ptr(self.k),
                                                self.state.h if self.state else None))

    def march(self, cam: Camera) -> None:
        camc = cam.c_struct()
        _lib.check(self.ctx.lib.fv_render_sparse(
            self.ctx.h, self.vol, C.byref(camc), self._light_ref(), C.byref(self._set),
            _lib.ptr(self.idx), _lib.ptr(self.k), self.h * self.w, None, None,
            self.state.h if self.state else None, None))

    def reconstruct(self, use_kernel_stage: bool = True) -> None:
        _lib.check(self.ctx.lib.fv_reconstruct(self.ctx.h, self.net_h, self.state.h, int(use_kernel_stage),
                                               _lib.ptr(self.rgb), None, None))

    def step(self, cam: Camera, fovea: FoveaConfig, frame: int, timed: bool = False):
        """One foveated frame on the device; returns per-phase ms when timed (syncs)."""
        s = self.ctx.stream
        if timed:
            self.ev[0].record(s)
        self.mask(fovea, frame)
        if timed:
            self.ev[1].record(s)
        self.march(cam)
        if timed:
            self.ev[2].record(s)
        self.reconstruct()
        if timed:
            self.ev[3].record(s)
            self.ev[3].synchronize()
            return (self.ev[0].elapsed_time(self.ev[1]), self.ev[1].elapsed_time(self.ev[2]),
                    self.ev[2].elapsed_time(self.ev[3]))
        return None

    def run_pipelined(self, frames, outs=None) -> None:
        """The frame loop through the C ABI's fv_frames: every frame replayed as one whole-frame CUDA
        graph (march t, then network t next to the mask of t+1). Frame t's image goes to outs[t]
        ((H,W,3) float32 CUDA tensors, entries may be None) or, by default, the last frame's into
        self.rgb. Launches only (stream-ordered on the pipeline's stream). FV_PIPE_PY=1: the Python
        stream-juggling loop below (separate mask / render / reconstruct calls)."""
        n = len(frames)
        if n == 0:
            return
        if outs is None:
            outs = [None] * (n - 1) + [self.rgb]
        if os.environ.get("FV_PIPE_PY", "0") != "1":
            cams = (_lib.FvCamera * n)(*[c.c_struct() for c, _, _ in frames])
            fovs = (_lib.FvFovea * n)(*[f.c_struct() for _, f, _ in frames])
            ids = (C.c_int * n)(*[int(j) for _, _, j in frames])
            ptrs = (C.c_void_p * n)(*[o.data_ptr() if o is not None else None for o in outs])
            _lib.check(self.ctx.lib.fv_frames(self.ctx.h, self.vol, self.net_h, self.state.h, n, cams,
                                              self._light_ref(), C.byref(self._set), fovs, ids, ptrs))
            return
        self._run_pipelined_py(frames, outs)

    def _run_pipelined_py(self, frames, outs) -> None:
        """Render frame t+1 (mask + march) on one stream while frame t reconstructs on another.

        `frames` is a sequence of (camera, fovea, frame index). The state's two input buffers
        alternate per frame (net.cu), so the only cross-stream dependencies are: frame t's
        network waits for frame t's render, and frame t's render waits for frame t-2's network
        (the last reader of the buffer it overwrites). Launches only; call sync_pipelined().
        """
        import torch

        if getattr(self, "_rctx", None) is None:
            # the network is the critical path: its stream gets the higher priority, so the marcher's
            # blocks fill the SMs the convs leave idle instead of delaying them
            prio = int(os.environ.get("FV_PIPE_PRIORITY", "1"))
            self._s_net = torch.cuda.Stream(device=self.ctx.device, priority=-1 if prio else 0)
            # FV_PIPE_OVERLAP=1: the render of frame t+1 on its own stream next to frame t's
            # network; by default one stream in frame order (see fv_frames in csrc/api.cu)
            overlap = os.environ.get("FV_PIPE_OVERLAP", "0") == "1"
            self._s_render = torch.cuda.Stream(device=self.ctx.device, priority=0) if overlap else self._s_net
            self._rctx = _lib.Context(self.ctx.device, stream=self._s_render)
            self._nctx = _lib.Context(self.ctx.device, stream=self._s_net)
            self._rctx.ensure_noise(self.ctx._noise_ref)
            self._vol_r = self.scene.volume.handle(self._rctx, self.scene.tf)
            # frame t+1's mask + compaction on a third (low-priority) stream as soon as frame t's march
            # has consumed the ray list, i.e. next to frame t's network (FV_MASK_AHEAD=0: in line)
            self._mask_ahead = os.environ.get("FV_MASK_AHEAD", "1") == "1"
            if self._mask_ahead:
                self._s_mask = torch.cuda.Stream(device=self.ctx.device, priority=0)
                self._mctx = _lib.Context(self.ctx.device, stream=self._s_mask)
                self._mctx.ensure_noise(self.ctx._noise_ref)
        s_r, s_n = self._s_render, self._s_net
        # both streams start after everything already queued on the pipeline's own stream
        start = torch.cuda.Event()
        start.record(self.ctx.stream)
        s_r.wait_event(start)
        s_n.wait_event(start)
        net_done = []
        ahead = self._mask_ahead
        masked = None
        if ahead:
            self._s_mask.wait_event(start)
            masked = self._mask_on(self._mctx, frames[0])
        for t, (cam, fovea, j) in enumerate(frames):
            if t >= 2:
                s_r.wait_event(net_done[t - 2])
            if ahead:
                s_r.wait_event(masked)
            else:
                self._mask_on(self._rctx, (cam, fovea, j))
            camc = cam.c_struct()
            _lib.check(self._rctx.lib.fv_render_sparse(
                self._rctx.h, self._vol_r, C.byref(camc), self._light_ref(), C.byref(self._set),
                _lib.ptr(self.idx), _lib.ptr(self.k), self.h * self.w, None, None, self.state.h, None))
            rendered = torch.cuda.Event()
            rendered.record(s_r)
            s_n.wait_event(rendered)
            _lib.check(self._nctx.lib.fv_reconstruct(self._nctx.h, self.net_h, self.state.h, 1,
                                                     _lib.ptr(outs[t] if outs[t] is not None else self.rgb),
                                                     None, None))
            done = torch.cuda.Event()
            done.record(s_n)
            net_done.append(done)
            if ahead and t + 1 < len(frames):
                # after frame t's reconstruct was enqueued: the state now points at frame t+1's input
                # buffer; the mask waits for frame t's march (the last reader of the ray list) and
                # frame t-1's network (the last reader of that buffer)
                self._s_mask.wait_event(rendered)
                if t >= 1:  # frame t-1's network read this input buffer (implied unless FV_PIPE_OVERLAP)
                    self._s_mask.wait_event(net_done[t - 1])
                masked = self._mask_on(self._mctx, frames[t + 1])
        # rejoin the pipeline's own stream
        self.ctx.stream.wait_event(net_done[-1])
        rj = torch.cuda.Event()
        rj.record(s_r)
        self.ctx.stream.wait_event(rj)

    def _mask_on(self, ctx, frame):
        """Enqueue one frame's mask + compaction on ctx's stream; returns the event after it."""
        import torch

        _, fovea, j = frame
        f = fovea.c_struct()
        _lib.check(ctx.lib.fv_mask_compact(ctx.h, int(j), self.h, self.w, C.byref(f), None, None,
                                           _lib.ptr(self.idx), _lib.ptr(self.k), self.state.h))
        ev = torch.cuda.Event()
        ev.record(ctx.stream)
        return ev

    def pipelined_contexts(self):
        return [c for c in (self.ctx, getattr(self, "_rctx", None), getattr(self, "_nctx", None),
                            getattr(self, "_mctx", None)) if c is not None]

    def dense(self, cam: Camera):
        """Dense baseline frame (render_full, renderer.py:211-222) into a device buffer."""
        import torch

        if self.dense_rgba is None:
            self.dense_rgba = torch.empty((self.h, self.w, 4), dtype=torch.float32, device="cuda")
        camc = cam.c_struct()
        _lib.check(self.ctx.lib.fv_render_full(self.ctx.h, self.vol, C.byref(camc), self._light_ref(),
                                               C.byref(self._set), _lib.ptr(self.dense_rgba), None, None))

    def frame_to_host(self, cam: Camera, fovea: FoveaConfig, frame: int, host_rgb: np.ndarray):
        """The whole frame through the C ABI's fv_frame with a host output buffer."""
        camc = cam.c_struct()
        f = fovea.c_struct()
        t = (C.c_double * 4)()
        _lib.check(self.ctx.lib.fv_frame(self.ctx.h, self.vol, self.net_h, self.state.h, C.byref(camc),
                                         self._light_ref(), C.byref(self._set), C.byref(f), int(frame),
                                         C.c_void_p(host_rgb.ctypes.data if isinstance(host_rgb, np.ndarray)
                                                    else host_rgb.data_ptr()), t))
        return tuple(t)

    def frames_to_host(self, frames, host_rgb) -> None:
        """A camera path through the C ABI's fv_frames: `frames` is a sequence of (camera, fovea,
        frame index); frame t's (H,W,3) float32 image lands in host_rgb[t % len(host_rgb)] (pinned
        torch tensors or NumPy arrays). Render t+1, reconstruct t and the copy of t-1 overlap on
        three streams; returns once every copy has landed."""
        n = len(frames)
        if n == 0:
            return
        cams = (_lib.FvCamera * n)(*[c.c_struct() for c, _, _ in frames])
        fovs = (_lib.FvFovea * n)(*[f.c_struct() for _, f, _ in frames])
        ids = (C.c_int * n)(*[int(j) for _, _, j in frames])

        def addr(b):
            return b.ctypes.data if isinstance(b, np.ndarray) else b.data_ptr()

        outs = (C.c_void_p * n)(*[addr(host_rgb[t % len(host_rgb)]) for t in range(n)])
        _lib.check(self.ctx.lib.fv_frames(self.ctx.h, self.vol, self.net_h, self.state.h, n, cams,
                                          self._light_ref(), C.byref(self._set), fovs, ids, outs))
