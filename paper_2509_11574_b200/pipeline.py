"""Per-frame mapping step (fuse -> raycast -> every delta_k frames: raycast the selected views
once, then `iterations` refine steps), driving libgps through the C ABI.

PAPER.md P:106 (per-frame fusion then raycast), P:138 (views raycast once per round)
(every 10 frames, 20 iterations), P:129 (keyframes).  Readings R-VIEW, R-VIEWS (schedule.py).
All compute is in libgps's kernels on one CUDA stream; this class only sequences calls and keeps
the device buffers.  Frames may be device tensors, or host tensors (copied in on the stream --
that is the end-to-end path).
"""
from __future__ import annotations

import numpy as np
import torch

from . import api as A
from . import schedule as Sch


class MappingPipeline:
    def __init__(self, cam: A.Camera, gaussians: A.Gaussians, volume: A.Volume, depth_scale: float,
                 render_cfg: A.RenderConfig | None = None, adam_cfg: A.AdamConfig | None = None,
                 delta_k: int = Sch.DELTA_K, iterations: int = Sch.ITERATIONS,
                 n_global: int = Sch.N_GLOBAL, n_local: int = Sch.N_LOCAL, seed: int = 0):
        self.cam, self.g, self.vol = cam, gaussians, volume
        self.depth_scale = float(depth_scale)
        self.rcfg = render_cfg or A.RenderConfig()
        self.adam = adam_cfg or A.AdamConfig()
        self.delta_k, self.iterations = delta_k, iterations
        self.n_global, self.n_local = n_global, n_local
        self.state = A.AdamState(gaussians)
        self.ras = A.Rasterizer(gaussians.n, cam, self.rcfg, n_views=1)
        self.kf = Sch.KeyframeSelector()
        self.rng = np.random.default_rng(seed)
        H, W = cam.height, cam.width
        dev = torch.device("cuda")
        self.depth = torch.empty((H, W), dtype=torch.float32, device=dev)   # D_t of the last frame
        self.color = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
        nv = n_global + n_local
        self.view_depth = [torch.empty((H, W), dtype=torch.float32, device=dev) for _ in range(nv)]
        self.view_color = [torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in range(nv)]
        self.frames = {}          # frame id -> (rgba device tensor, R, t) for keyframes and the interval
        self.interval = []
        self.last_frame = None
        self.last_loss = None
        self.copy_stream = torch.cuda.Stream()
        self.rounds = 0
        self.iterations_run = 0

    def _device(self, x: torch.Tensor) -> torch.Tensor:
        """Host frames are uploaded on a dedicated copy stream (pinned memory -> async), so frame
        k+1's upload overlaps frame k's kernels; the compute stream waits on an event."""
        if x.is_cuda:
            return x
        compute = torch.cuda.current_stream()
        with torch.cuda.stream(self.copy_stream):
            d = x.to("cuda", non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        compute.wait_event(ev)
        d.record_stream(compute)
        return d

    def process_frame(self, k: int, depth: torch.Tensor, rgba: torch.Tensor, R, t, refine: bool = True):
        depth = self._device(depth)
        rgba = self._device(rgba)
        self.vol.fuse(self.cam, R, t, depth, self.depth_scale, rgba)
        self.vol.raycast(self.cam, R, t, self.depth, self.color)
        self.last_frame = k
        is_kf = self.kf.offer(k, R, t)
        self.interval.append(k)
        self.frames[k] = (rgba, np.asarray(R, np.float32), np.asarray(t, np.float32))
        if refine and Sch.is_round_frame(k, self.delta_k):
            self.refine_round()
        if len(self.interval) >= self.delta_k or Sch.is_round_frame(k, self.delta_k):
            self.interval = []
        # keep device frames only for keyframes and the current interval
        keep = set(self.kf.keyframes) | set(self.interval)
        for f in [f for f in self.frames if f not in keep]:
            del self.frames[f]
        return is_kf

    def snapshot(self):
        """Complete mapping state (device copies of the volume, Gaussians and Adam moments, plus
        the host bookkeeping) for replaying a window of the sequence."""
        import copy
        return {"vol": self.vol.clone(), "g": self.g.clone(), "m": self.state.m.clone(), "v": self.state.v.clone(),
                "step": self.state.step, "kf": (list(self.kf.keyframes), copy.deepcopy(self.kf._last)),
                "frames": dict(self.frames), "interval": list(self.interval), "last_frame": self.last_frame,
                "rng": copy.deepcopy(self.rng.bit_generator.state), "rounds": self.rounds,
                "iterations_run": self.iterations_run}

    def restore(self, s):
        self.vol.copy_from(s["vol"])
        for k in A.FIELDS:
            getattr(self.g, k).copy_(getattr(s["g"], k))
            getattr(self.state.m, k).copy_(getattr(s["m"], k))
            getattr(self.state.v, k).copy_(getattr(s["v"], k))
        self.state.step = s["step"]
        self.kf.keyframes, self.kf._last = list(s["kf"][0]), s["kf"][1]
        self.frames, self.interval, self.last_frame = dict(s["frames"]), list(s["interval"]), s["last_frame"]
        self.rng.bit_generator.state = s["rng"]
        self.rounds, self.iterations_run = s["rounds"], s["iterations_run"]

    def refine_round(self):
        views_ids = Sch.select_views(self.kf.keyframes, self.interval, self.rng, self.n_global, self.n_local)
        views = []
        for j, f in enumerate(views_ids):
            rgba, R, t = self.frames[f]
            if f == self.last_frame:
                # the frame just fused was raycast against this very volume: same result
                views.append(A.View(self.cam, R, t, self.depth, self.color, rgba))
                continue
            self.vol.raycast(self.cam, R, t, self.view_depth[j], self.view_color[j])
            views.append(A.View(self.cam, R, t, self.view_depth[j], self.view_color[j], rgba))
        for i in range(self.iterations):
            v = views[Sch.view_for_iteration(i, len(views))]
            self.last_loss = self.ras.refine_step(self.g, self.state, [v], self.adam)
        self.rounds += 1
        self.iterations_run += self.iterations
        return views_ids
