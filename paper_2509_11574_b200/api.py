"""Torch-facing API over libgps (the C ABI of include/gps.h).

Torch supplies device memory and streams only; every step of the mapping path runs in
libgps.so's sm_100a kernels.  Functions take torch tensors (device unless noted), pass their
pointers and the current CUDA stream to the C ABI, and raise GPSError on a non-OK status.

Paper: GPS-SLAM, arXiv 2509.11574.  gps_fuse/gps_raycast: Sec. 3.2.1 and
Sec. 3.1 first pass; gps_render: Eqs. 1-4; gps_refine_step: Eq. 7,
Adam with App. C learning rates.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N

_L = N.load()


def _stream(stream=None) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def c(self) -> N.gps_intrinsics:
        return N.gps_intrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


def pose_struct(R, t) -> N.gps_pose:
    R = np.asarray(R, np.float32).reshape(9)
    t = np.asarray(t, np.float32).reshape(3)
    return N.gps_pose((C.c_float * 9)(*R.tolist()), (C.c_float * 3)(*t.tolist()))


def pose_tensor(R, t, out: torch.Tensor | None = None) -> torch.Tensor:
    """A gps_pose in device memory (f32[12]: R row-major, t) for the *_dpose entry points."""
    h = torch.from_numpy(np.concatenate([np.asarray(R, np.float32).reshape(9), np.asarray(t, np.float32).reshape(3)]))
    if out is None:
        return h.cuda()
    out.copy_(h)
    return out


def _dpose(pose: torch.Tensor) -> int:
    assert pose.is_cuda and pose.dtype == torch.float32 and pose.numel() == 12 and pose.is_contiguous()
    return _ptr(pose)


# ---------------------------------------------------------------------------------------------
# volume
# ---------------------------------------------------------------------------------------------
VOXEL_DTYPE = np.dtype([("tsdf", "<f4"), ("rgbw", "u1", (4,))])


class Volume:
    """Voxel-block hash volume owned by libgps (gps_volume_*)."""

    def __init__(self, voxel_size=0.005, mu=None, w_max=100, depth_min=0.1, depth_max=10.0,
                 max_blocks=1 << 18, hash_slots=1 << 20, dense_bounds=None, stream=None):
        """dense_bounds: optional ((x0, y0, z0), (x1, y1, z1)) in metres covered by the dense
        block-index grid (an accelerator for the raycast; results do not depend on it)."""
        mu = 4 * voxel_size if mu is None else mu
        org, dims = (0, 0, 0), (0, 0, 0)
        if dense_bounds is not None:
            bs = 8 * voxel_size
            lo = [int(np.floor(c / bs)) - 1 for c in dense_bounds[0]]
            hi = [int(np.ceil(c / bs)) + 1 for c in dense_bounds[1]]
            org, dims = tuple(lo), tuple(h - l for l, h in zip(lo, hi))
        self.cfg = N.gps_volume_config(voxel_size, mu, w_max, depth_min, depth_max, int(max_blocks),
                                       int(hash_slots), (C.c_int32 * 3)(*org), (C.c_int32 * 3)(*dims))
        h = C.c_void_p()
        N.check("gps_volume_create", _L.gps_volume_create(C.byref(self.cfg), _stream(stream), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            torch.cuda.synchronize()
            _L.gps_volume_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, stream=None):
        N.check("gps_volume_reset", _L.gps_volume_reset(self.h, _stream(stream)))

    def copy_from(self, other: "Volume", stream=None):
        """Device-to-device copy of another volume's complete state (identical configs)."""
        N.check("gps_volume_copy", _L.gps_volume_copy(self.h, other.h, _stream(stream)))

    def clone(self, stream=None) -> "Volume":
        v = Volume.__new__(Volume)
        v.cfg = N.gps_volume_config.from_buffer_copy(self.cfg)
        h = C.c_void_p()
        N.check("gps_volume_create", _L.gps_volume_create(C.byref(v.cfg), _stream(stream), C.byref(h)))
        v.h = h
        v.copy_from(self, stream)
        return v

    def fuse(self, cam: Camera, R, t, depth: torch.Tensor, depth_scale: float, rgba: torch.Tensor,
             stream=None):
        """depth: u16/i16 [H,W] raw sensor units; rgba: u8 [H,W,4].  CPU tensors are copied to
        the device first (that copy is part of an end-to-end measurement)."""
        if not depth.is_cuda or not rgba.is_cuda:
            # the copies run on the stream the fuse runs on, so the caching allocator cannot
            # hand the temporaries to another stream before the kernels have read them
            if stream is None:
                s = torch.cuda.current_stream()
            elif isinstance(stream, torch.cuda.Stream):
                s = stream
            else:
                s = torch.cuda.ExternalStream(_stream(stream))
            with torch.cuda.stream(s):
                if not depth.is_cuda:
                    depth = depth.cuda(non_blocking=True)
                if not rgba.is_cuda:
                    rgba = rgba.cuda(non_blocking=True)
        assert depth.element_size() == 2 and depth.numel() == cam.width * cam.height
        assert rgba.dtype == torch.uint8 and rgba.numel() == 4 * cam.width * cam.height
        N.check("gps_fuse", _L.gps_fuse(self.h, C.byref(cam.c()), C.byref(pose_struct(R, t)), _ptr(depth),
                                        float(depth_scale), _ptr(rgba), _stream(stream)))

    def fuse_dpose(self, cam: Camera, pose: torch.Tensor, depth: torch.Tensor, depth_scale: float,
                   rgba: torch.Tensor, stream=None):
        """gps_fuse_dpose: as fuse, the pose read on the device from `pose` (pose_tensor layout)."""
        assert depth.is_cuda and rgba.is_cuda
        assert depth.element_size() == 2 and depth.numel() == cam.width * cam.height
        assert rgba.dtype == torch.uint8 and rgba.numel() == 4 * cam.width * cam.height
        N.check("gps_fuse_dpose", _L.gps_fuse_dpose(self.h, C.byref(cam.c()), _dpose(pose), _ptr(depth),
                                                    float(depth_scale), _ptr(rgba), _stream(stream)))

    def raycast_dpose(self, cam: Camera, pose: torch.Tensor, depth_out, color_out, vertex_out=None, stream=None):
        """gps_raycast_dpose: as raycast, the pose read on the device."""
        N.check("gps_raycast_dpose", _L.gps_raycast_dpose(self.h, C.byref(cam.c()), _dpose(pose), _ptr(depth_out),
                                                          _ptr(color_out), _ptr(vertex_out), _stream(stream)))
        return depth_out, color_out, vertex_out

    def raycast(self, cam: Camera, R, t, depth_out=None, color_out=None, vertex_out=None,
                want_vertex=False, stream=None):
        dev = torch.device("cuda")
        if depth_out is None:
            depth_out = torch.empty((cam.height, cam.width), dtype=torch.float32, device=dev)
        if color_out is None:
            color_out = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev)
        if want_vertex and vertex_out is None:
            vertex_out = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev)
        N.check("gps_raycast", _L.gps_raycast(self.h, C.byref(cam.c()), C.byref(pose_struct(R, t)),
                                              _ptr(depth_out), _ptr(color_out), _ptr(vertex_out),
                                              _stream(stream)))
        return depth_out, color_out, vertex_out

    def fuse_raycast(self, cam: Camera, R, t, depth: torch.Tensor, depth_scale: float, rgba: torch.Tensor,
                     depth_out, color_out, vertex_out=None, graph: bool = True, stream=None):
        """gps_fuse_raycast: fuse the frame, then raycast it from the same pose, in one call (one
        CUDA graph with graph=True on a created stream).  Device frames only."""
        assert depth.is_cuda and rgba.is_cuda
        assert depth.element_size() == 2 and depth.numel() == cam.width * cam.height
        assert rgba.dtype == torch.uint8 and rgba.numel() == 4 * cam.width * cam.height
        N.check("gps_fuse_raycast",
                _L.gps_fuse_raycast(self.h, C.byref(cam.c()), C.byref(pose_struct(R, t)), _ptr(depth),
                                    float(depth_scale), _ptr(rgba), _ptr(depth_out), _ptr(color_out),
                                    _ptr(vertex_out), int(graph), _stream(stream)))
        return depth_out, color_out, vertex_out

    def stats(self, stream=None):
        nb, bud, nv, vt, ut = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        st = _L.gps_volume_stats_sync(self.h, _stream(stream), C.byref(nb), C.byref(bud), C.byref(nv), C.byref(vt),
                                      C.byref(ut))
        return {"n_blocks": nb.value, "budget": bud.value, "n_visible": nv.value, "visible_total": vt.value,
                "updated_total": ut.value, "status": N.STATUS[st]}

    def export_blocks(self, with_voxels=True, stream=None):
        """(coords i32[n,3], voxels structured [n,512] (tsdf f32, rgbw u8[4]) or None), any order."""
        cap = int(self.cfg.max_blocks)
        coords = torch.empty((cap, 3), dtype=torch.int32, device="cuda")
        vox = torch.empty((cap, 512, 2), dtype=torch.int32, device="cuda") if with_voxels else None
        n = C.c_int64()
        N.check("gps_debug_export_blocks_sync",
                _L.gps_debug_export_blocks_sync(self.h, _stream(stream), _ptr(coords), _ptr(vox), cap, C.byref(n)))
        k = min(n.value, cap)
        c = coords[:k].cpu().numpy()
        v = None
        if with_voxels:
            v = vox[:k].cpu().numpy().view(VOXEL_DTYPE).reshape(k, 512)
        return c, v

    def apron_mismatches(self, stream=None) -> int:
        """Apron cells (the + face copies of the tsdf plane) that differ from their owner voxels;
        0 after every fuse (debug; synchronises)."""
        n = C.c_int64()
        N.check("gps_debug_apron_check_sync", _L.gps_debug_apron_check_sync(self.h, _stream(stream), C.byref(n)))
        return n.value

    def hash_mismatches(self, stream=None) -> int:
        """Violations of the hash / pool / neighbour-table invariants (gps_debug_hash_check_sync);
        0 after every fuse (debug; synchronises)."""
        n = C.c_int64()
        N.check("gps_debug_hash_check_sync", _L.gps_debug_hash_check_sync(self.h, _stream(stream), C.byref(n)))
        return n.value

    def raycast_footprint(self, cam: Camera, R, t, stream=None) -> int:
        """Number of distinct tsdf voxels a raycast from (R, t) reads (debug; synchronises)."""
        n = C.c_int64()
        N.check("gps_debug_raycast_footprint_sync",
                _L.gps_debug_raycast_footprint_sync(self.h, C.byref(cam.c()), C.byref(pose_struct(R, t)),
                                                   _stream(stream), C.byref(n)))
        return n.value

    def export_visible(self, stream=None):
        cap = int(self.cfg.max_blocks)
        coords = torch.empty((cap, 3), dtype=torch.int32, device="cuda")
        n = C.c_int64()
        N.check("gps_debug_export_visible_sync",
                _L.gps_debug_export_visible_sync(self.h, _stream(stream), _ptr(coords), cap, C.byref(n)))
        return coords[:min(n.value, cap)].cpu().numpy()


# ---------------------------------------------------------------------------------------------
# Gaussians, optimiser state, rasteriser
# ---------------------------------------------------------------------------------------------
FIELDS = ("xyz", "log_scale", "rot", "opacity_raw", "sh")


class Gaussians:
    """Caller-owned SoA parameter arrays (float32, contiguous, CUDA).  The arrays hold `capacity`
    Gaussians (default n); the public attributes are views of the first n rows, so Gaussian
    adding / removal (gps_add_gaussians_sync / gps_remove_gaussians_sync) change n in place."""

    def __init__(self, n: int, sh_degree: int, device="cuda", tensors: dict | None = None,
                 capacity: int | None = None):
        self.sh_degree = int(sh_degree)
        n = int(n)
        cap = max(int(capacity if capacity is not None else n), n)
        nc = (sh_degree + 1) ** 2
        self._shapes = {"xyz": (3,), "log_scale": (3,), "rot": (4,), "opacity_raw": (), "sh": (nc * 3,)}
        self._store = {}
        for k in FIELDS:
            buf = torch.zeros((cap,) + self._shapes[k], dtype=torch.float32, device=device)
            if tensors is not None:
                v = torch.as_tensor(np.asarray(tensors[k], np.float32)).reshape((n,) + self._shapes[k])
                buf[:n].copy_(v.to(device))
            self._store[k] = buf
        self.capacity = cap
        self.set_n(n)

    def set_n(self, n: int):
        if n > self.capacity:
            raise ValueError("n exceeds capacity")
        self.n = int(n)
        self._c = None  # the cached C struct carries n
        for k in FIELDS:
            setattr(self, k, self._store[k][:self.n])

    @staticmethod
    def from_dict(d: dict, device="cuda", capacity: int | None = None) -> "Gaussians":
        return Gaussians(int(np.asarray(d["xyz"]).shape[0]), int(d["sh_degree"]), device, d, capacity)

    def zeros_like(self) -> "Gaussians":
        return Gaussians(self.n, self.sh_degree, self.xyz.device, capacity=self.capacity)

    def c(self) -> N.gps_gaussians:
        # cached: the storage never moves and n changes only through set_n (host cost per call)
        if getattr(self, "_c", None) is None:
            self._c = N.gps_gaussians(self.n, self.sh_degree, *(C.c_void_p(self._store[k].data_ptr()) for k in FIELDS))
        return self._c

    def to_numpy(self) -> dict:
        out = {k: getattr(self, k).detach().cpu().numpy() for k in FIELDS}
        out["sh_degree"] = self.sh_degree
        return out

    def clone(self) -> "Gaussians":
        g = Gaussians(self.n, self.sh_degree, self.xyz.device, capacity=self.capacity)
        for k in FIELDS:
            getattr(g, k).copy_(getattr(self, k))
        return g


class AdamState:
    def __init__(self, g: Gaussians):
        self.m = g.zeros_like()
        self.v = g.zeros_like()
        self.step = 0


@dataclass
class RenderConfig:
    eps_depth: float = 0.02          # R-EPS  ("small positive threshold")
    alpha_min: float = 1.0 / 255
    near_z: float = 0.2              # R-NEAR
    lowpass: float = 0.3             # R-LOWPASS
    tile: int = 16
    tile_depth_precull: int = 1
    max_pairs: int = 0
    sort_free: int = 0               # 1: the paper's sort-free rendering
    backward: int = 0                # 0: the renderer's own scheme, 1: warp per entry, 2: thread per group

    def c(self) -> N.gps_render_config:
        return N.gps_render_config(self.eps_depth, self.alpha_min, self.near_z, self.lowpass, self.tile,
                                   self.tile_depth_precull, self.max_pairs, self.sort_free, self.backward)


@dataclass
class AdamConfig:
    lr_xyz: float = 1.6e-4
    lr_sh0: float = 2.5e-3
    lr_shrest: float = 5e-4
    lr_opacity: float = 5e-2
    lr_scale: float = 5e-3
    lr_rot: float = 1e-3
    beta1: float = 0.9         # R-ADAM
    beta2: float = 0.999
    eps: float = 1e-15

    def c(self) -> N.gps_adam_config:
        return N.gps_adam_config(self.lr_xyz, self.lr_sh0, self.lr_shrest, self.lr_opacity, self.lr_scale,
                                 self.lr_rot, self.beta1, self.beta2, self.eps)


@dataclass
class View:
    cam: Camera
    R: np.ndarray
    t: np.ndarray
    sdf_depth: torch.Tensor
    sdf_color: torch.Tensor
    target_rgba: torch.Tensor

    def c(self) -> N.gps_view:
        # built once: a View is not modified after its first use (the pipeline makes new ones)
        if getattr(self, "_c", None) is None:
            self._c = N.gps_view(self.cam.c(), pose_struct(self.R, self.t), _ptr(self.sdf_depth),
                                 _ptr(self.sdf_color), _ptr(self.target_rgba))
        return self._c


class Rasterizer:
    """Owns the device workspace of gps_render / gps_refine_step for up to n Gaussians."""

    def __init__(self, n: int, cam: Camera, cfg: RenderConfig | None = None, n_views: int = 1):
        self.cfg = cfg or RenderConfig()
        self.n, self.cam, self.n_views = n, cam, n_views
        size = _L.gps_refine_workspace_size(n, C.byref(cam.c()), C.byref(self.cfg.c()), n_views)
        if size == 0:
            raise ValueError("bad rasteriser configuration")
        self.ws = torch.empty(size, dtype=torch.uint8, device="cuda")
        self.loss = torch.zeros(1, dtype=torch.float32, device="cuda")

    def reserve(self, n: int):
        """Grow the workspace for up to n Gaussians (after Gaussian adding)."""
        if n <= self.n:
            return
        size = _L.gps_refine_workspace_size(n, C.byref(self.cam.c()), C.byref(self.cfg.c()), self.n_views)
        self.ws = torch.empty(size, dtype=torch.uint8, device="cuda")
        self.n = n

    def render(self, g: Gaussians, cam: Camera, R, t, sdf_depth, sdf_color, target_rgba=None,
               out_color=None, out_weight=None, stream=None):
        if out_color is None:
            out_color = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda")
        if out_weight is None:
            out_weight = torch.empty((cam.height, cam.width), dtype=torch.float32, device="cuda")
        loss = self.loss if target_rgba is not None else None
        N.check("gps_render", _L.gps_render(C.byref(g.c()), C.byref(cam.c()), C.byref(pose_struct(R, t)),
                                            _ptr(sdf_depth), _ptr(sdf_color), _ptr(target_rgba),
                                            C.byref(self.cfg.c()), _ptr(self.ws), self.ws.numel(),
                                            _ptr(out_color), _ptr(out_weight), _ptr(loss), _stream(stream)))
        return out_color, out_weight, loss

    def refine_step(self, g: Gaussians, state: AdamState, views: list[View], adam: AdamConfig | None = None,
                    grad_out: Gaussians | None = None, stream=None):
        adam = adam or AdamConfig()
        arr = (N.gps_view * len(views))(*[v.c() for v in views])
        st = N.gps_adam_state(state.m.c(), state.v.c(), state.step)
        gc = g.c()
        go = grad_out.c() if grad_out is not None else None
        key = (id(adam), tuple(adam.__dict__.values()), tuple(self.cfg.__dict__.values()))
        if getattr(self, "_ckey", None) != key:  # the config structs, rebuilt only when they change
            self._ckey, self._cc = key, (self.cfg.c(), adam.c())
        N.check("gps_refine_step",
                _L.gps_refine_step(C.byref(gc), C.byref(st), arr, len(views), C.byref(self._cc[0]),
                                   C.byref(self._cc[1]), _ptr(self.ws), self.ws.numel(), _ptr(self.loss),
                                   C.byref(go) if go is not None else None, _stream(stream)))
        state.step = st.step
        return self.loss

    def refine_round(self, g: Gaussians, state: AdamState, views: list[View], iter_views,
                     adam: AdamConfig | None = None, graph: bool = True, stream=None):
        """n_iter refine_step iterations in one call (gps_refine_round): iteration i uses the views
        views[j] for j in iter_views[i] (a sequence of index sequences of equal length); with
        graph=True the round runs as one CUDA graph (on a created stream)."""
        adam = adam or AdamConfig()
        rows = [list(r) for r in iter_views]
        per = len(rows[0]) if rows else 1
        if any(len(r) != per for r in rows):
            raise ValueError("every iteration must use the same number of views")
        flat = [j for r in rows for j in r]
        idx = (C.c_int32 * max(len(flat), 1))(*flat)
        arr = (N.gps_view * len(views))(*[v.c() for v in views])
        st = N.gps_adam_state(state.m.c(), state.v.c(), state.step)
        gc = g.c()
        key = (id(adam), tuple(adam.__dict__.values()), tuple(self.cfg.__dict__.values()))
        if getattr(self, "_ckey", None) != key:
            self._ckey, self._cc = key, (self.cfg.c(), adam.c())
        N.check("gps_refine_round",
                _L.gps_refine_round(C.byref(gc), C.byref(st), arr, len(views), idx, per, len(rows),
                                    C.byref(self._cc[0]), C.byref(self._cc[1]), _ptr(self.ws), self.ws.numel(),
                                    _ptr(self.loss), int(graph), _stream(stream)))
        state.step = st.step
        return self.loss

    def stats(self, stream=None):
        K, cap, nv = C.c_int64(), C.c_int64(), C.c_int64()
        st = _L.gps_render_stats_sync(_ptr(self.ws), _stream(stream), C.byref(K), C.byref(cap), C.byref(nv))
        return {"pairs": K.value, "capacity": cap.value, "n_visible": nv.value, "status": N.STATUS[st]}

    def pair_counts(self, g: Gaussians, cam: Camera, R, t, sdf_depth, sdf_color, stream=None):
        """(evaluated, accepted) pixel-entry pairs of one instrumented forward (debug; syncs)."""
        e, a = C.c_int64(), C.c_int64()
        N.check("gps_debug_render_counts_sync",
                _L.gps_debug_render_counts_sync(C.byref(g.c()), C.byref(cam.c()), C.byref(pose_struct(R, t)),
                                                _ptr(sdf_depth), _ptr(sdf_color), C.byref(self.cfg.c()),
                                                _ptr(self.ws), self.ws.numel(), C.byref(e), C.byref(a),
                                                _stream(stream)))
        return e.value, a.value

    def lists(self, stream=None):
        """(values u32[K], ranges u32[n_tiles, 2]) of the last render."""
        cam = self.cam
        tiles = -(-cam.width // self.cfg.tile) * -(-cam.height // self.cfg.tile)
        K = C.c_int64()
        N.check("gps_debug_render_lists_sync",
                _L.gps_debug_render_lists_sync(_ptr(self.ws), _stream(stream), None, 0, None, C.byref(K)))
        vals = torch.empty(max(K.value, 1), dtype=torch.int32, device="cuda")
        ranges = torch.empty((tiles, 2), dtype=torch.int32, device="cuda")
        N.check("gps_debug_render_lists_sync",
                _L.gps_debug_render_lists_sync(_ptr(self.ws), _stream(stream), _ptr(vals), K.value, _ptr(ranges),
                                               C.byref(K)))
        return (vals[:K.value].cpu().numpy().view(np.uint32), ranges.cpu().numpy().view(np.uint32))


def adam_step(g: Gaussians, state: AdamState, grad: Gaussians, adam: AdamConfig | None = None, stream=None):
    adam = adam or AdamConfig()
    st = N.gps_adam_state(state.m.c(), state.v.c(), state.step)
    N.check("gps_adam_step", _L.gps_adam_step(C.byref(g.c()), C.byref(st), C.byref(grad.c()), C.byref(adam.c()),
                                              _stream(stream)))
    state.step = st.step


# ---------------------------------------------------------------------------------------------
# Gaussian adding and removal
# ---------------------------------------------------------------------------------------------
@dataclass
class AddConfig:
    delta_c: float = 0.05      # Eq. 6
    delta_w: float = 4.0       # Eq. 6
    sample_frac: float = 0.25
    opacity_init: float = 0.5
    scale_max: float = 0.1     # App. A
    knn_cell: float = 0.01     # kNN grid cell (accelerator only)
    seed: int = 0              # R-SAMPLE

    def c(self) -> N.gps_add_config:
        return N.gps_add_config(self.delta_c, self.delta_w, self.sample_frac, self.opacity_init, self.scale_max,
                                self.knn_cell, self.seed & 0xFFFFFFFF, 0)


@dataclass
class RemoveConfig:
    sigma_min: float = 0.005   # Eq. 8
    scale_max: float = 0.1
    scale_min: float = 0.003

    def c(self) -> N.gps_remove_config:
        return N.gps_remove_config(self.sigma_min, self.scale_max, self.scale_min, 0)


def vertex_normals(cam: Camera, R, t, sdf_depth: torch.Tensor, vertex: torch.Tensor, out=None, stream=None):
    """N* from the raycast vertex map (gps_vertex_normals, R-NORMAL)."""
    if out is None:
        out = torch.empty_like(vertex)
    N.check("gps_vertex_normals", _L.gps_vertex_normals(C.byref(cam.c()), C.byref(pose_struct(R, t)), _ptr(sdf_depth),
                                                        _ptr(vertex), _ptr(out), _stream(stream)))
    return out


def vertex_normals_dpose(cam: Camera, pose: torch.Tensor, sdf_depth: torch.Tensor, vertex: torch.Tensor, out,
                         stream=None):
    """gps_vertex_normals_dpose: the camera centre read from a device pose."""
    N.check("gps_vertex_normals_dpose",
            _L.gps_vertex_normals_dpose(C.byref(cam.c()), _dpose(pose), _ptr(sdf_depth), _ptr(vertex), _ptr(out),
                                        _stream(stream)))
    return out


_ws_cache: dict = {}


def _ws(key, size):
    t = _ws_cache.get(key)
    if t is None or t.numel() < size:
        t = torch.empty(size, dtype=torch.uint8, device="cuda")
        _ws_cache[key] = t
    return t


def add_gaussians(g: Gaussians, state: AdamState, cam: Camera, sdf_depth, vertex, normal, cstar, weight,
                  target_rgba, cfg: AddConfig | None = None, stream=None):
    """Gaussian adding (gps_add_gaussians_sync): appends to g (up to its capacity) and zeroes
    the new Gaussians' Adam moments; returns (added, candidates).  Synchronises."""
    cfg = cfg or AddConfig()
    ws = _ws("add", _L.gps_add_workspace_size(C.byref(cam.c())))
    st = N.gps_adam_state(state.m.c(), state.v.c(), state.step)
    gc = g.c()
    added, cand = C.c_int64(), C.c_int64()
    N.check("gps_add_gaussians_sync",
            _L.gps_add_gaussians_sync(C.byref(gc), g.capacity, C.byref(st), C.byref(cam.c()), _ptr(sdf_depth),
                                      _ptr(vertex), _ptr(normal), _ptr(cstar), _ptr(weight), _ptr(target_rgba),
                                      C.byref(cfg.c()), _ptr(ws), ws.numel(), C.byref(added), C.byref(cand),
                                      _stream(stream)))
    for x in (g, state.m, state.v):
        x.set_n(gc.n)
    return added.value, cand.value


def remove_gaussians(g: Gaussians, state: AdamState, cfg: RemoveConfig | None = None, stream=None) -> int:
    """Gaussian removal (gps_remove_gaussians_sync): stable in-place compaction of g and its Adam
    moments; returns the number removed.  Synchronises."""
    cfg = cfg or RemoveConfig()
    ws = _ws("remove", _L.gps_remove_workspace_size(g.n, g.sh_degree))
    st = N.gps_adam_state(state.m.c(), state.v.c(), state.step)
    gc = g.c()
    removed = C.c_int64()
    N.check("gps_remove_gaussians_sync",
            _L.gps_remove_gaussians_sync(C.byref(gc), C.byref(st), C.byref(cfg.c()), _ptr(ws), ws.numel(),
                                         C.byref(removed), _stream(stream)))
    for x in (g, state.m, state.v):
        x.set_n(gc.n)
    return removed.value


# ---------------------------------------------------------------------------------------------
# camera tracking
# ---------------------------------------------------------------------------------------------
@dataclass
class IcpConfig:
    levels: int = 3
    iters: tuple = (10, 5, 4)      # finest -> coarsest
    dist_max: float = 0.1
    angle_max_deg: float = 30.0
    depth_min: float = 0.1
    depth_max: float = 10.0
    eps: float = 1e-6
    min_inlier_frac: float = 0.1
    fallback: bool = True          # R-ICP-FAIL: a frame that does not converge keeps its initial pose
    min_inlier_px_frac: float = 0.05  # R-ICP-FAIL: converged needs inliers >= this fraction of the pixels
    min_pivot_ratio: float = 1e-3     # R-ICP-FAIL: ... and a well-conditioned last system
    filter_radius: int = 0            # R-ICP-FILT: bilateral pre-filter of the tracking depth (0 = off;
                                      # MappingPipeline tracks with 3)
    filter_sigma_s: float = 4.5
    filter_sigma_r: float = 0.03

    def c(self) -> N.gps_icp_config:
        it = list(self.iters) + [1] * (4 - len(self.iters))
        return N.gps_icp_config(self.levels, (C.c_int32 * 4)(*it), self.dist_max, self.angle_max_deg,
                                self.depth_min, self.depth_max, self.eps, self.min_inlier_frac,
                                int(self.fallback), self.min_inlier_px_frac, self.min_pivot_ratio,
                                int(self.filter_radius), self.filter_sigma_s, self.filter_sigma_r)


def track(cam: Camera, depth: torch.Tensor, depth_scale: float, model_vertex: torch.Tensor,
          model_normal: torch.Tensor, R_model, t_model, R_init, t_init, cfg: IcpConfig | None = None,
          stream=None) -> dict:
    """Frame-to-model ICP (gps_track_sync, Eq. 5): returns {"R", "t" (fp64 numpy), "converged",
    "degenerate", "inlier_frac", "inliers", "steps", "energy"}.  Synchronises."""
    cfg = cfg or IcpConfig()
    ws = _ws("track", _L.gps_track_workspace_size(C.byref(cam.c()), cfg.levels))
    out = N.gps_track_result()
    N.check("gps_track_sync",
            _L.gps_track_sync(C.byref(cam.c()), _ptr(depth), float(depth_scale), _ptr(model_vertex),
                              _ptr(model_normal), C.byref(pose_struct(R_model, t_model)),
                              C.byref(pose_struct(R_init, t_init)), C.byref(cfg.c()), _ptr(ws), ws.numel(),
                              C.byref(out), _stream(stream)))
    return {"R": np.array(out.R64[:], np.float64).reshape(3, 3), "t": np.array(out.t64[:], np.float64),
            "T": (np.array(out.T.R[:], np.float32).reshape(3, 3), np.array(out.T.t[:], np.float32)),
            "converged": bool(out.converged), "degenerate": bool(out.degenerate), "inlier_frac": out.inlier_frac,
            "inliers": out.inliers, "steps": out.steps, "energy": out.energy, "pivot_ratio": out.pivot_ratio}


TRACK_RESULT_BYTES = C.sizeof(N.gps_track_result)


def track_async(cam: Camera, depth: torch.Tensor, depth_scale: float, model_vertex: torch.Tensor,
                model_normal: torch.Tensor, pose_model: torch.Tensor, pose_init: torch.Tensor, pose_out: torch.Tensor,
                result_out: torch.Tensor | None = None, cfg: IcpConfig | None = None, stream=None, ws=None,
                pose_fail: torch.Tensor | None = None):
    """gps_track_async: ICP with every pose in device memory (pose_tensor layout) and no
    synchronisation; result_out (nullable) is a u8[TRACK_RESULT_BYTES] device tensor that
    receives the gps_track_result (decode with track_result())."""
    cfg = cfg or IcpConfig()
    if ws is None:
        ws = _ws("track", _L.gps_track_workspace_size(C.byref(cam.c()), cfg.levels))
    if result_out is not None:
        assert result_out.is_cuda and result_out.numel() >= TRACK_RESULT_BYTES
    N.check("gps_track_async",
            _L.gps_track_async(C.byref(cam.c()), _ptr(depth), float(depth_scale), _ptr(model_vertex),
                               _ptr(model_normal), _dpose(pose_model), _dpose(pose_init),
                               None if pose_fail is None else _dpose(pose_fail), C.byref(cfg.c()), _ptr(ws),
                               ws.numel(), _dpose(pose_out), _ptr(result_out), _stream(stream)))
    return pose_out


def pose_extrapolate(pose_a: torch.Tensor, pose_b: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """gps_pose_extrapolate: out <- T_b (T_a^-1 T_b), the constant-velocity prediction (device)."""
    N.check("gps_pose_extrapolate", _L.gps_pose_extrapolate(_dpose(pose_a), _dpose(pose_b), _dpose(out),
                                                            _stream(stream)))
    return out


def track_result(raw) -> dict:
    """Decode a gps_track_result copied to the host (bytes / u8 tensor) as track() returns it."""
    b = bytes(raw.cpu().numpy().tobytes() if isinstance(raw, torch.Tensor) else raw)[:TRACK_RESULT_BYTES]
    out = N.gps_track_result.from_buffer_copy(b)
    return {"R": np.array(out.R64[:], np.float64).reshape(3, 3), "t": np.array(out.t64[:], np.float64),
            "T": (np.array(out.T.R[:], np.float32).reshape(3, 3), np.array(out.T.t[:], np.float32)),
            "converged": bool(out.converged), "degenerate": bool(out.degenerate), "inlier_frac": out.inlier_frac,
            "inliers": out.inliers, "steps": out.steps, "energy": out.energy, "pivot_ratio": out.pivot_ratio}


def check_word() -> tuple[int, bool]:
    """(OR of the checked build's failed-bound bits since the last call, whether the loaded library
    is the checked build); synchronises the device (gps_debug_check_word_sync)."""
    w, c = C.c_int64(), C.c_int32()
    N.check("gps_debug_check_word_sync", _L.gps_debug_check_word_sync(C.byref(w), C.byref(c)))
    return w.value, bool(c.value)
