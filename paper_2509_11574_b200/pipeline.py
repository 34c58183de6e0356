"""Per-frame mapping step (fuse -> raycast -> every delta_k frames: raycast the selected views
once, then `iterations` refine steps), driving libgps through the C ABI.

PAPER.md P:106 (per-frame fusion then raycast), P:138 (views raycast once per round)
(every 10 frames, 20 iterations), P:129 (keyframes).  Readings R-VIEW, R-VIEWS (schedule.py).
All compute is in libgps's kernels (fusion and raycasts on the caller's stream, refinement on a
second stream when overlap=True); this class only sequences calls and keeps the device buffers.
Frames may be device tensors, or host tensors (copied in on a copy stream -- that is the
end-to-end path).  On a created (non-default) stream each frame's fuse + raycast and each round's
iterations run as CUDA graphs (gps_fuse_raycast, gps_refine_round; graphs=False: direct
launches); the host is held at most max_frames_ahead frames ahead of the device.
"""
from __future__ import annotations

import collections
import contextlib
import ctypes as C
import dataclasses
import time

import numpy as np
import torch

from . import api as A
from . import schedule as Sch


class MappingPipeline:
    """overlap=True runs each round's refinement on a second stream while the following frames
    are fused and raycast on the caller's stream -- the paper's two parallel threads (P:116,
    "the SDF ... and the 3D Gaussian ... are executed in parallel").  The data dependencies are
    those of the serial schedule: a round reads only its views' raycasts (taken at the round
    frame), its targets and the Gaussians, none of which the fusion stream writes; view
    buffers are double-buffered across rounds, and a round's buffer set is reused only after the
    refinement that read it (two rounds earlier) has finished.  join() makes the caller's stream
    wait for the refinement stream."""

    def __init__(self, cam: A.Camera, gaussians: A.Gaussians, volume: A.Volume, depth_scale: float,
                 render_cfg: A.RenderConfig | None = None, adam_cfg: A.AdamConfig | None = None,
                 delta_k: int = Sch.DELTA_K, iterations: int = Sch.ITERATIONS,
                 n_global: int = Sch.N_GLOBAL, n_local: int = Sch.N_LOCAL, seed: int = 0,
                 overlap: bool = True, refine_priority: int = -1, manage_gaussians: bool = False,
                 add_cfg: A.AddConfig | None = None, remove_cfg: A.RemoveConfig | None = None,
                 all_views_per_iteration: bool = False, track: bool = False,
                 icp_cfg: A.IcpConfig | None = None, graphs: bool = True, max_frames_ahead: int = 20,
                 frame_graphs: bool | None = None, view_priority: int | None = None,
                 upload_reserve_mb: int = 1024):
        self.cam, self.g, self.vol = cam, gaussians, volume
        self.graphs = graphs  # each refinement round as one CUDA graph (gps_refine_round)
        # each frame's fuse + raycast as one CUDA graph (gps_fuse_raycast; default: as `graphs`)
        self.frame_graphs = graphs if frame_graphs is None else frame_graphs
        # the host enqueues at most max_frames_ahead frames beyond the device's fusion stream (0:
        # unbounded): bounds the frames in flight, so the caching allocator stops growing
        self.max_ahead = max_frames_ahead
        self._inflight = collections.deque()
        self.host_wait_s = 0.0  # host time spent waiting on that bound
        # device memory for the host-frame uploads, reserved in the copy stream's allocator pool
        # at the first upload: a cudaMalloc while the GPU is busy blocked the host for 14-85 ms
        # (measured), so the uploads must be served from cached blocks
        self.upload_reserve_mb = upload_reserve_mb
        self._reserved = False
        self.depth_scale = float(depth_scale)
        self.rcfg = render_cfg or A.RenderConfig()
        self.adam = adam_cfg or A.AdamConfig()
        self.delta_k, self.iterations = delta_k, iterations
        self.n_global, self.n_local = n_global, n_local
        self.state = A.AdamState(gaussians)
        # workspace sized for the Gaussians' capacity: adding never reallocates it mid-stream
        # R-VIEW: one view per iteration; all_views_per_iteration: every iteration renders all the
        # round's views and sums their gradients (SPEC S:471 variant)
        self.all_views = all_views_per_iteration
        self.ras = A.Rasterizer(gaussians.capacity, cam, self.rcfg,
                                n_views=(n_global + n_local) if all_views_per_iteration else 1)
        # camera tracking (Eq. 5): every frame after the first is
        # tracked against the previous frame's raycast maps, and its tracked pose is the one fused
        # The tracked pose stays on the device: ICP writes it (gps_track_async) into a ring slot
        # that fusion, raycast and normals read (the *_dpose forms) and the next frame's ICP
        # starts from; a copy goes to pinned host memory, read lazily (keyframe selection and the
        # round's views need it only at round frames), so a frame costs no host round trip.
        self.tracking = track
        self.icp_cfg = icp_cfg or A.IcpConfig(filter_radius=3)  # R-ICP-FILT on the tracking depth
        self._track_log = []
        self._pending = []       # frames whose keyframe offer waits for their host pose, in order
        self._last_pose = None
        self._pose_dev = None    # device pose (f32[12]) of the last fused frame, tracking mode
        self._pose_prev = None   # ... and of the frame before it (constant-velocity prediction)
        self.poses = {}          # frame -> host (R, t) as fused, tracking mode (filled by _resolve)
        # Gaussian adding / removal
        self.manage = manage_gaussians
        self.add_cfg = add_cfg or A.AddConfig()
        self.remove_cfg = remove_cfg or A.RemoveConfig()
        self.added_total = 0
        self.removed_total = 0
        self._removal_pending = False
        self.kf = Sch.KeyframeSelector()
        self.rng = np.random.default_rng(seed)
        H, W = cam.height, cam.width
        dev = torch.device("cuda")
        # D_t / C_t of the last frame (aliases a view buffer when that frame is a round view)
        self._fdepth = torch.empty((H, W), dtype=torch.float32, device=dev)
        self._fcolor = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
        self.depth, self.color = self._fdepth, self._fcolor
        nv = n_global + n_local
        # adding inputs of a round frame (its D_t, C_t, V*, N*) and the second-pass render, one set
        # per view-buffer set: written by the fusion stream at the round frame, read by the
        # refinement stream in that round, rewritten two rounds later (after _set_free)
        mk = lambda *shape: [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(2)]
        if track:
            self.t_vertex = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
            self.t_normal = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
            self._model = None  # (V*, N*) of the previous frame
            rb = (A.TRACK_RESULT_BYTES + 15) // 16 * 16
            self._ring = 64
            self._res_dev = torch.zeros((self._ring, rb), dtype=torch.uint8, device=dev)
            self._res_host = torch.zeros((self._ring, rb), dtype=torch.uint8, pin_memory=True)
            self._slot = 0
            self._pred = torch.empty(12, dtype=torch.float32, device=dev)
            self._track_ws = torch.empty(A._L.gps_track_workspace_size(C.byref(cam.c()), self.icp_cfg.levels),
                                         dtype=torch.uint8, device=dev)
        if manage_gaussians:
            self.r_depth, self.r_color, self.vertex, self.normal = mk(H, W), mk(H, W, 3), mk(H, W, 3), mk(H, W, 3)
            self._add_color, self._add_weight = mk(H, W, 3), mk(H, W)
        nsets = 2
        self.view_depth = [[torch.empty((H, W), dtype=torch.float32, device=dev) for _ in range(nv)]
                           for _ in range(nsets)]
        self.view_color = [[torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in range(nv)]
                           for _ in range(nsets)]
        self.frames = {}          # frame id -> (rgba device tensor, R, t) for keyframes and the interval
        self.interval = []
        self.last_frame = None
        self.last_loss = None
        self.copy_stream = torch.cuda.Stream()
        self.overlap = overlap  # may be switched between rounds
        # the refinement rounds are the longer of the two streams' work: give them the higher
        # scheduling priority so fusion and raycasts fill the SMs around them
        self.refine_stream = torch.cuda.Stream(priority=refine_priority)
        # view_priority: the round's view raycasts on a third stream of that priority (ordered after
        # the round frame's fusion; the next frames' fusion waits for them), else on the fusion stream
        self.view_stream = torch.cuda.Stream(priority=view_priority) if view_priority is not None else None
        self._set_free = [None] * nsets   # event: the refinement that last read buffer set s is done
        self._refine_done = None
        self.rounds = 0
        self.iterations_run = 0

    def _upload(self, x: torch.Tensor):
        """Start the H2D copy of a pinned host tensor on the copy stream; (device tensor, event)."""
        if not self._reserved:
            self._reserved = True
            if self.upload_reserve_mb > 0:
                with torch.cuda.stream(self.copy_stream):
                    torch.empty(self.upload_reserve_mb << 20, dtype=torch.uint8, device="cuda")
        with torch.cuda.stream(self.copy_stream):
            d = x.to("cuda", non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        return d, ev

    def _device(self, x: torch.Tensor) -> torch.Tensor:
        """Host frames are uploaded on a dedicated copy stream (pinned memory -> async); a frame
        announced by the previous call's `prefetch` is already in flight.  The compute stream
        waits on the copy's event."""
        if x.is_cuda:
            return x
        pre = self._prefetched.pop(id(x), None) if hasattr(self, "_prefetched") else None
        if pre is not None and pre[0] is x:
            d, ev = pre[1], pre[2]
        else:
            d, ev = self._upload(x)
        compute = torch.cuda.current_stream()
        compute.wait_event(ev)
        d.record_stream(compute)
        return d

    def prefetch(self, *host_tensors):
        """Start uploading the next frame's host tensors now (its process_frame call picks them up)."""
        if not hasattr(self, "_prefetched"):
            self._prefetched = {}
        for x in host_tensors:
            if x is not None and not x.is_cuda and id(x) not in self._prefetched:
                d, ev = self._upload(x)
                self._prefetched[id(x)] = (x, d, ev)

    def process_frame(self, k: int, depth: torch.Tensor, rgba: torch.Tensor, R, t, refine: bool = True,
                      prefetch=None):
        """One frame of the mapping step.  `prefetch`: the next frame's (depth, rgba) host tensors,
        whose upload then overlaps this frame's kernels."""
        if self.max_ahead and len(self._inflight) >= self.max_ahead:
            t0 = time.perf_counter()
            self._inflight.popleft().synchronize()
            self.host_wait_s += time.perf_counter() - t0
        depth = self._device(depth)
        rgba = self._device(rgba)
        if prefetch is not None:
            self.prefetch(*prefetch)
        dpose = None
        if self.tracking:
            if self._model is not None:
                dpose = self._track(k, depth)
            else:  # the first frame: its given pose starts the trajectory
                dpose = self._pose_dev = A.pose_tensor(R, t)
                self._pending.append((k, None, (np.asarray(R, np.float32), np.asarray(t, np.float32))))
            self.vol.fuse_dpose(self.cam, dpose, depth, self.depth_scale, rgba)
            is_kf = None  # decided when the pose is read back (_resolve)
            self.frames[k] = (rgba, None, None)
        else:
            # fused together with its raycast below (gps_fuse_raycast: one CUDA graph per frame)
            self._last_pose = (np.asarray(R, np.float32), np.asarray(t, np.float32))
            is_kf = self.kf.offer(k, R, t)
            self.frames[k] = (rgba, np.asarray(R, np.float32), np.asarray(t, np.float32))
        self.last_frame = k
        self.interval.append(k)
        round_now = refine and Sch.is_round_frame(k, self.delta_k)
        if round_now and self.tracking:
            self._resolve()  # the keyframes and the views' host poses (waits for this frame's ICP)
            R, t = self._last_pose
        views_ids = None
        self.depth, self.color = self._fdepth, self._fcolor
        want_v = round_now and self.manage
        if round_now:
            views_ids = Sch.select_views(self.kf.keyframes, self.interval, self.rng, self.n_global, self.n_local)
            s = self.rounds % len(self.view_depth)
            self._wait_set(s)
            if want_v:
                # the round frame's raycast also feeds Gaussian adding: into the round's set
                self.depth, self.color = self.r_depth[s], self.r_color[s]
            elif k in views_ids:
                # the frame just fused is a view: its per-frame raycast is the view's
                j = views_ids.index(k)
                self.depth, self.color = self.view_depth[s][j], self.view_color[s][j]
        vert = self.vertex[s] if want_v else (self.t_vertex if self.tracking else None)
        if self.tracking:
            self.vol.raycast_dpose(self.cam, dpose, self.depth, self.color, vert)
            nrm = self.normal[s] if want_v else self.t_normal
            A.vertex_normals_dpose(self.cam, dpose, self.depth, vert, nrm)
            self._model = (vert, nrm)
        else:
            self.vol.fuse_raycast(self.cam, R, t, depth, self.depth_scale, rgba, self.depth, self.color,
                                  vertex_out=vert, graph=self.frame_graphs)
            if want_v:
                A.vertex_normals(self.cam, R, t, self.depth, self.vertex[s], out=self.normal[s])
        if round_now:
            self._refine_round(views_ids, add_frame=(k, rgba, R, t, s) if self.manage else None)
        if len(self.interval) >= self.delta_k or Sch.is_round_frame(k, self.delta_k):
            self.interval = []
        if not self._pending:
            self._drop_frames()
        if self.max_ahead:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self._inflight.append(ev)
        return is_kf

    def _drop_frames(self):
        """Keep device frames only for keyframes and the current interval."""
        keep = set(self.kf.keyframes) | set(self.interval)
        for f in [f for f in self.frames if f not in keep]:
            del self.frames[f]

    def _track(self, k, depth):
        """ICP of frame k against the previous frame's maps, from the previous frame's device pose
        (gps_track_async); the result record is copied to pinned memory for _resolve."""
        if len(self._pending) >= self._ring - 1:
            self._resolve()  # the oldest pending slot is about to be reused
        i = self._slot
        self._slot = (i + 1) % self._ring
        raw = self._res_dev[i]
        pose = raw[:48].view(torch.float32)  # gps_track_result.T is its first member
        # the ICP starts from the previous frame's pose, whose camera is also the association's (Eq. 5);
        # a frame whose ICP fails gets the constant-velocity prediction from the two previous
        # frames instead (R-ICP-FAIL); with no prediction yet (the second frame) the iterate stands
        cfg = self.icp_cfg
        fail = None
        if self._pose_prev is not None:
            fail = A.pose_extrapolate(self._pose_prev, self._pose_dev, self._pred)
        elif cfg.fallback:
            cfg = dataclasses.replace(cfg, fallback=False)
        A.track_async(self.cam, depth, self.depth_scale, self._model[0], self._model[1], self._pose_dev,
                      self._pose_dev, pose, raw, cfg, ws=self._track_ws, pose_fail=fail)
        self._pose_prev = self._pose_dev
        self._res_host[i].copy_(raw, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._pending.append((k, (i, ev), None))
        self._pose_dev = pose
        return pose

    def _resolve(self):
        """Read back the pending tracked poses (waiting only for the last one's ICP), and make the
        deferred keyframe offers in frame order."""
        if not self._pending:
            return
        for k, dev, host in self._pending:
            if dev is not None:
                i, ev = dev
                ev.synchronize()
                res = A.track_result(self._res_host[i])
                self._track_log.append(res)
                host = res["T"]  # the fused pose (the iterate, or the prediction on failure)
            R, t = host
            self.poses[k] = host
            self.kf.offer(k, R, t)
            if k in self.frames:
                self.frames[k] = (self.frames[k][0], R, t)
            self._last_pose = host
        self._pending = []
        self._drop_frames()

    @property
    def last_pose(self):
        """Host (R, t) of the last fused frame (tracking mode: waits for its ICP)."""
        self._resolve()
        return self._last_pose

    @property
    def track_log(self):
        self._resolve()
        return self._track_log

    def _wait_set(self, s: int):
        ev = self._set_free[s]
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def join(self, stream=None):
        """Order `stream` (default: the current stream) after all refinement issued so far."""
        if self._refine_done is not None:
            (stream or torch.cuda.current_stream()).wait_event(self._refine_done)

    def loss_to(self, dst: torch.Tensor):
        """Asynchronous copy of the last refinement loss into dst (e.g. pinned host memory),
        ordered on the refinement stream so the fusion stream never waits for it."""
        if self.last_loss is None:
            return
        with torch.cuda.stream(self.refine_stream if self.overlap else torch.cuda.current_stream()):
            dst.copy_(self.last_loss, non_blocking=True)

    def snapshot(self):
        """Complete mapping state (device copies of the volume, Gaussians and Adam moments, plus
        the host bookkeeping) for replaying a window of the sequence."""
        import copy
        self.join()
        self._resolve()
        return {"vol": self.vol.clone(), "g": self.g.clone(), "m": self.state.m.clone(), "v": self.state.v.clone(),
                "step": self.state.step, "kf": (list(self.kf.keyframes), copy.deepcopy(self.kf._last)),
                "frames": dict(self.frames), "interval": list(self.interval), "last_frame": self.last_frame,
                "rng": copy.deepcopy(self.rng.bit_generator.state), "rounds": self.rounds,
                "iterations_run": self.iterations_run, "removal_pending": self._removal_pending,
                "added_total": self.added_total, "removed_total": self.removed_total,
                "track": ((self._model[0].clone(), self._model[1].clone(), self._pose_dev.clone(), self._last_pose,
                           None if self._pose_prev is None else self._pose_prev.clone())
                          if self.tracking and self._model is not None else None)}

    def restore(self, s):
        self.join()
        self._resolve()
        self.vol.copy_from(s["vol"])
        for x in (self.g, self.state.m, self.state.v):
            x.set_n(s["g"].n)
        for k in A.FIELDS:
            getattr(self.g, k).copy_(getattr(s["g"], k))
            getattr(self.state.m, k).copy_(getattr(s["m"], k))
            getattr(self.state.v, k).copy_(getattr(s["v"], k))
        self.state.step = s["step"]
        self.kf.keyframes, self.kf._last = list(s["kf"][0]), s["kf"][1]
        self.frames, self.interval, self.last_frame = dict(s["frames"]), list(s["interval"]), s["last_frame"]
        self.rng.bit_generator.state = s["rng"]
        self.rounds, self.iterations_run = s["rounds"], s["iterations_run"]
        self._removal_pending = s["removal_pending"]
        self.added_total, self.removed_total = s["added_total"], s["removed_total"]
        if self.tracking and s["track"] is not None:
            self._pending = []
            self.t_vertex.copy_(s["track"][0])
            self.t_normal.copy_(s["track"][1])
            self._model = (self.t_vertex, self.t_normal)
            self._pose_dev = s["track"][2].clone()
            self._pose_prev = None if s["track"][4] is None else s["track"][4].clone()
            self._last_pose = s["track"][3]
        if True:  # the refinement stream must see the restored state
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self.refine_stream.wait_event(ev)

    def refine_round(self):
        """A round at the current point of the sequence (views chosen now; the last frame's
        raycast is recomputed into the round's buffers)."""
        self._resolve()
        views_ids = Sch.select_views(self.kf.keyframes, self.interval, self.rng, self.n_global, self.n_local)
        self._wait_set(self.rounds % len(self.view_depth))
        return self._refine_round(views_ids, reuse_last=False)

    def _manage(self, rs, add_frame):
        """On the refinement stream, before the round's iterations: the previous round's Gaussian
        removal (Eq. 8: "after each Gaussian optimization" -- nothing reads the
        Gaussians in between, so deferring it to here is the same sequence), then Gaussian adding
        for the round frame (Eq. 6) from its raycast V*, N* and a second-pass render
        with the existing Gaussians.  Both synchronise (the new count is host state)."""
        if self._removal_pending:
            self.removed_total += A.remove_gaussians(self.g, self.state, self.remove_cfg, stream=rs)
            self._removal_pending = False
        k, rgba, R, t, s = add_frame
        self.ras.render(self.g, self.cam, R, t, self.r_depth[s], self.r_color[s], None, self._add_color[s],
                        self._add_weight[s], stream=rs)
        cfg = A.AddConfig(**{**self.add_cfg.__dict__, "seed": (self.add_cfg.seed * 1000003 + k) & 0xFFFFFFFF})
        added, _ = A.add_gaussians(self.g, self.state, self.cam, self.r_depth[s], self.vertex[s], self.normal[s],
                                   self._add_color[s], self._add_weight[s], rgba, cfg, stream=rs)
        self.added_total += added

    def _refine_round(self, views_ids, reuse_last: bool = True, add_frame=None):
        s = self.rounds % len(self.view_depth)
        views = []
        cur = torch.cuda.current_stream()
        vs = self.view_stream if self.overlap else None
        if vs is not None:
            vs.wait_stream(cur)  # after the round frame's fusion
        with torch.cuda.stream(vs) if vs is not None else contextlib.nullcontext():
            for j, f in enumerate(views_ids):
                rgba, R, t = self.frames[f]
                if reuse_last and f == self.last_frame:
                    # the frame just fused was raycast against this very volume: same result
                    views.append(A.View(self.cam, R, t, self.depth, self.color, rgba))
                    continue
                self.vol.raycast(self.cam, R, t, self.view_depth[s][j], self.view_color[s][j])
                views.append(A.View(self.cam, R, t, self.view_depth[s][j], self.view_color[s][j], rgba))
        if vs is not None:
            cur.wait_stream(vs)  # the next frames' fusion writes the volume the raycasts read
        if self.overlap:
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream())
            rs = self.refine_stream
            rs.wait_event(ready)
            for v in views:
                v.target_rgba.record_stream(rs)
            if add_frame is not None:
                add_frame[1].record_stream(rs)
        else:
            rs = torch.cuda.current_stream()
            self.join(rs)  # after any refinement still running from an overlapped round
        with torch.cuda.stream(rs):
            if add_frame is not None:
                self._manage(rs, add_frame)
            self.last_view = views[-1]
            self.last_views = list(views)
            if self.all_views:
                order = [list(range(len(views)))] * self.iterations
            else:
                order = [[Sch.view_for_iteration(i, len(views))] for i in range(self.iterations)]
            # the round's iterations in one library call, replayed as one CUDA graph
            self.last_loss = self.ras.refine_round(self.g, self.state, views, order, self.adam,
                                                   graph=self.graphs, stream=rs)
            done = torch.cuda.Event()
            done.record(rs)
        if self.manage:
            self._removal_pending = True
        self._set_free[s] = done
        self._refine_done = done
        self.rounds += 1
        self.iterations_run += self.iterations
        return views_ids
