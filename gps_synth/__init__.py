"""Seeded synthetic RGB-D inputs for the GPS-SLAM mapping step.

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU oracle.  It
holds no arithmetic of the method (no fusion, raycast, projection or blending): it ray-traces
analytic primitives (planes, boxes, spheres) to produce sensor-like frames, and draws
Gaussian parameters, exactly as DESIGN.md §5 ("input recipe") describes.

Configs (BASELINE.json ``configs``; shapes from SURVEY.md §8(d)):
  cfg1  64x48 plane + sphere, identity pose, 1k Gaussians, 1 refine iteration (parity case)
  cfg2  TUM-shaped 640x480, depth/5000, Kinect-v1 noise
  cfg3  Replica-shaped 1200x680, exact depth (scale 6553.5), 137,200 Gaussians
  cfg4  Azure-Kinect-shaped 1280x720, depth in mm, ToF noise, 200k Gaussians (headline)

Everything is torch (CPU or CUDA); parity tests generate on CPU and copy to the device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

# ----------------------------------------------------------------------------------------------
# configurations
# ----------------------------------------------------------------------------------------------


@dataclass
class SynthConfig:
    name: str
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    depth_scale: float          # raw u16 units per metre
    n_frames: int
    n_gaussians: int
    scene: str                  # "plane_sphere" | "room"
    room: tuple = (6.0, 5.0, 3.0)
    n_objects: int = 8
    noise: str = "none"         # "none" | "kinect1" | "tof"
    dropout: float = 0.0
    range_max: float = 10.0
    range_min: float = 0.1
    step_m: float = 0.0067      # camera path length per frame
    scale_mm: tuple = (3.0, 20.0)
    sh_degree: int = 3
    seed: int = 0
    # volume sizing
    voxel_size: float = 0.005
    max_blocks: int = 1 << 18
    hash_slots: int = 1 << 20
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "cfg1": SynthConfig("cfg1", 64, 48, 60.0, 60.0, 31.5, 23.5, 1e4, 1, 1000, "plane_sphere",
                        scale_mm=(3.0, 15.0), seed=0, max_blocks=512, hash_slots=1024),
    "cfg2": SynthConfig("cfg2", 640, 480, 525.0, 525.0, 319.5, 239.5, 5000.0, 300, 50_000, "room",
                        room=(4.0, 4.0, 2.6), n_objects=5, noise="kinect1", dropout=0.02,
                        range_max=4.5, step_m=0.008, seed=2, max_blocks=1 << 18,
                        hash_slots=1 << 20),
    "cfg3": SynthConfig("cfg3", 1200, 680, 600.0, 600.0, 599.5, 339.5, 6553.5, 2000, 137_200,
                        "room", room=(6.0, 5.0, 3.0), n_objects=8, noise="none", seed=3,
                        max_blocks=1 << 19, hash_slots=1 << 21),
    "cfg4": SynthConfig("cfg4", 1280, 720, 605.0, 605.0, 639.5, 359.5, 1000.0, 3000, 200_000,
                        "room", room=(8.0, 6.0, 2.8), n_objects=10, noise="tof", dropout=0.06,
                        range_min=0.25, range_max=5.5, seed=4, max_blocks=1 << 19,
                        hash_slots=1 << 21),
    # NEXT-4: ScanNet++-shaped, 1752x1168 ("2.2x ... standard"), a DSLR-like
    # clean depth (no sensor noise), fx scaled from cfg4's field of view; intrinsics invented
    "scannetpp": SynthConfig("scannetpp", 1752, 1168, 828.0, 828.0, 875.5, 583.5, 1000.0, 3000, 200_000,
                             "room", room=(8.0, 6.0, 2.8), n_objects=10, noise="none", dropout=0.0,
                             range_min=0.25, range_max=8.0, seed=6, max_blocks=1 << 19, hash_slots=1 << 21),
}


def scene_bounds(cfg: "SynthConfig", margin: float = 0.5):
    """Axis-aligned bounds (metres) that contain the scene, for the optional dense block grid."""
    if cfg.scene == "plane_sphere":
        return ((-0.5, -0.5, -0.1), (0.5, 0.5, 0.6))
    X, Y, Z = cfg.room
    return ((-margin, -margin, -margin), (X + margin, Y + margin, Z + margin))


def get_config(name: str, **over) -> SynthConfig:
    import dataclasses
    return dataclasses.replace(CONFIGS[name], **over)


# ----------------------------------------------------------------------------------------------
# scene: analytic primitives with procedural albedo
# ----------------------------------------------------------------------------------------------


@dataclass
class Prim:
    kind: str                 # "plane" | "sphere" | "box_in" | "box_out"
    a: np.ndarray             # plane: point; sphere: centre; box: min corner
    b: np.ndarray             # plane: unit normal; sphere: (r,0,0); box: max corner
    color0: np.ndarray
    color1: np.ndarray
    tex: str                  # "checker" | "noise" | "ramp" | "stripes"
    tex_scale: float
    waves: np.ndarray         # (k, 3) wave vectors for "noise"
    phases: np.ndarray        # (k, 3) phase per channel


class Scene:
    def __init__(self, prims: list[Prim], light=(0.3, -0.4, 0.85), ambient=0.35, specular=0.0):
        self.prims = prims
        l = np.asarray(light, np.float64)
        self.light = l / np.linalg.norm(l)
        self.ambient = ambient
        self.specular = specular

    # -- intersection ---------------------------------------------------------------------
    @staticmethod
    def _hit(p: Prim, o, d):
        """ray o + t d (o: (3,), d: (n,3) unit, float64 torch) -> (t (n,), normal (n,3))."""
        dev = d.device
        big = torch.full((d.shape[0],), float("inf"), dtype=d.dtype, device=dev)
        if p.kind == "plane":
            n = torch.as_tensor(p.b, dtype=d.dtype, device=dev)
            a = torch.as_tensor(p.a, dtype=d.dtype, device=dev)
            den = d @ n
            t = ((a - o) @ n) / den
            ok = (den.abs() > 1e-12) & (t > 1e-6)
            nn = n.expand_as(d)
            nn = torch.where((den > 0)[:, None], -nn, nn)
            return torch.where(ok, t, big), nn
        if p.kind == "sphere":
            c = torch.as_tensor(p.a, dtype=d.dtype, device=dev)
            r = float(p.b[0])
            oc = o - c
            bq = d @ oc
            cq = float(oc @ oc) - r * r
            disc = bq * bq - cq
            sq = torch.sqrt(disc.clamp_min(0))
            t0 = -bq - sq
            t1 = -bq + sq
            t = torch.where(t0 > 1e-6, t0, t1)
            ok = (disc >= 0) & (t > 1e-6)
            t = torch.where(ok, t, big)
            pt = o + t.clamp(max=1e6)[:, None] * d
            nn = (pt - c) / r
            return t, nn
        lo = torch.as_tensor(p.a, dtype=d.dtype, device=dev)
        hi = torch.as_tensor(p.b, dtype=d.dtype, device=dev)
        inv = 1.0 / torch.where(d.abs() < 1e-12, torch.full_like(d, 1e-12), d)
        ta = (lo - o) * inv
        tb = (hi - o) * inv
        tmin = torch.minimum(ta, tb)
        tmax = torch.maximum(ta, tb)
        tn, an = tmin.max(dim=1)
        tf, af = tmax.min(dim=1)
        if p.kind == "box_in":  # camera inside: the far wall
            t = torch.where(tf > 1e-6, tf, big)
            axis = af
            sgn = torch.where(d.gather(1, axis[:, None])[:, 0] > 0, -1.0, 1.0)
        else:
            ok = (tn <= tf) & (tn > 1e-6)
            t = torch.where(ok, tn, big)
            axis = an
            sgn = torch.where(d.gather(1, axis[:, None])[:, 0] > 0, -1.0, 1.0)
        nn = torch.zeros_like(d)
        nn.scatter_(1, axis[:, None], sgn.to(d.dtype)[:, None])
        return t, nn

    def _albedo(self, p: Prim, pts):
        dev, dt = pts.device, pts.dtype
        c0 = torch.as_tensor(p.color0, dtype=dt, device=dev)
        c1 = torch.as_tensor(p.color1, dtype=dt, device=dev)
        if p.tex == "checker":
            k = torch.floor(pts / p.tex_scale).sum(dim=1).remainder(2.0)
            return torch.where(k[:, None] > 0.5, c1, c0)
        if p.tex == "stripes":
            k = torch.floor(pts[:, 0] / p.tex_scale).remainder(2.0)
            return torch.where(k[:, None] > 0.5, c1, c0)
        if p.tex == "ramp":
            s = (pts[:, 0] - p.a[0]) / (2 * p.b[0]) + 0.5
            return c0 + (c1 - c0) * s.clamp(0, 1)[:, None]
        w = torch.as_tensor(p.waves, dtype=dt, device=dev)
        ph = torch.as_tensor(p.phases, dtype=dt, device=dev)
        arg = pts @ w.T  # (n,k)
        v = torch.stack([torch.sin(arg + ph[:, ch]).mean(dim=1) for ch in range(3)], dim=1)
        mix = (0.5 + 0.5 * v).clamp(0, 1)
        return c0 + (c1 - c0) * mix

    def trace(self, o, d):
        """Nearest hit over all primitives: (t, normal, albedo, valid), float64 torch."""
        best_t = None
        best_n = None
        best_i = None
        for i, p in enumerate(self.prims):
            t, n = self._hit(p, o, d)
            if best_t is None:
                best_t, best_n = t, n
                best_i = torch.zeros_like(t, dtype=torch.long)
            else:
                closer = t < best_t
                best_t = torch.where(closer, t, best_t)
                best_n = torch.where(closer[:, None], n, best_n)
                best_i = torch.where(closer, torch.full_like(best_i, i), best_i)
        valid = torch.isfinite(best_t)
        pts = o + torch.where(valid, best_t, torch.zeros_like(best_t))[:, None] * d
        alb = torch.zeros_like(pts)
        for i, p in enumerate(self.prims):
            sel = valid & (best_i == i)
            if sel.any():
                alb[sel] = self._albedo(p, pts[sel])
        return best_t, best_n, alb, valid, pts

    def shade(self, albedo, normal, d, exposure=1.0):
        l = torch.as_tensor(self.light, dtype=albedo.dtype, device=albedo.device)
        lam = (normal @ l).abs()
        c = albedo * (self.ambient + (1 - self.ambient) * lam)[:, None]
        if self.specular > 0:
            h = l - d
            h = h / h.norm(dim=1, keepdim=True)
            c = c + self.specular * (normal * h).sum(dim=1).abs().pow(30)[:, None]
        return (c * exposure).clamp(0, 1)


def _rand_color(rng, lo=0.15, hi=0.9):
    return rng.uniform(lo, hi, size=3)


def _noise_tex(rng, k=6, fmin=3.0, fmax=40.0):
    dirs = rng.normal(size=(k, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    freq = np.exp(rng.uniform(np.log(fmin), np.log(fmax), size=(k, 1)))
    return dirs * freq, rng.uniform(0, 2 * np.pi, size=(k, 3))


def make_scene(cfg: SynthConfig) -> Scene:
    rng = np.random.default_rng(1000 + cfg.seed)
    if cfg.scene == "plane_sphere":
        w, ph = _noise_tex(rng)
        plane = Prim("plane", np.array([0, 0, 0.30]), np.array([0, 0, -1.0]),
                     np.array([0.85, 0.8, 0.7]), np.array([0.2, 0.25, 0.45]), "checker", 0.01, w, ph)
        sphere = Prim("sphere", np.array([0.03, -0.02, 0.22]), np.array([0.04, 0, 0]),
                      np.array([0.9, 0.2, 0.1]), np.array([0.1, 0.6, 0.9]), "ramp", 1.0, w, ph)
        return Scene([plane, sphere], light=(0.0, 0.0, -1.0), ambient=0.5)
    X, Y, Z = cfg.room
    prims = []
    w, ph = _noise_tex(rng)
    prims.append(Prim("box_in", np.array([0.0, 0.0, 0.0]), np.array([X, Y, Z]),
                      _rand_color(rng, 0.5, 0.9), _rand_color(rng, 0.2, 0.6), "noise", 1.0, w, ph))
    for k in range(cfg.n_objects):
        w, ph = _noise_tex(rng)
        tex = ["checker", "noise", "stripes"][k % 3]
        c0, c1 = _rand_color(rng), _rand_color(rng)
        if k % 4 == 3:
            r = rng.uniform(0.15, 0.4)
            c = np.array([rng.uniform(r + 0.3, X - r - 0.3), rng.uniform(r + 0.3, Y - r - 0.3),
                          rng.uniform(r, 1.2)])
            prims.append(Prim("sphere", c, np.array([r, 0, 0]), c0, c1, "noise", 1.0, w, ph))
        else:
            sx, sy, sz = rng.uniform(0.3, 1.2), rng.uniform(0.3, 1.0), rng.uniform(0.3, 1.1)
            # furniture along the walls, leaving the middle free for the camera path
            side = k % 4
            if side == 0:
                x0, y0 = rng.uniform(0.1, X - sx - 0.1), 0.05
            elif side == 1:
                x0, y0 = X - sx - 0.05, rng.uniform(0.1, Y - sy - 0.1)
            else:
                x0, y0 = rng.uniform(0.1, X - sx - 0.1), Y - sy - 0.05
            prims.append(Prim("box_out", np.array([x0, y0, 0.0]), np.array([x0 + sx, y0 + sy, sz]),
                              c0, c1, tex, rng.uniform(0.03, 0.12), w, ph))
    return Scene(prims, specular=0.08 if cfg.noise == "tof" else 0.0)


# ----------------------------------------------------------------------------------------------
# camera path
# ----------------------------------------------------------------------------------------------


def look_pose(eye, target, up=(0.0, 0.0, 1.0)):
    """camera->world pose with camera x right, y down, z forward (R columns = camera axes)."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    x = np.cross(f, np.asarray(up, np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    R = np.stack([x, y, f], axis=1)
    return R.astype(np.float32), eye.astype(np.float32)


def trajectory(cfg: SynthConfig, n: int, start: int = 0):
    """Smooth seeded path: an ellipse around the room centre at ~1.4 m height, looking at a
    slowly rotating point on the far side (handheld-like bob and yaw wobble)."""
    if cfg.scene == "plane_sphere":
        return [(np.eye(3, dtype=np.float32), np.zeros(3, np.float32)) for _ in range(n)]
    X, Y, Z = cfg.room
    rng = np.random.default_rng(2000 + cfg.seed)
    a, b = 0.3 * X, 0.3 * Y
    rho = 0.5 * (a + b)
    ph0 = rng.uniform(0, 2 * np.pi)
    poses = []
    for k in range(start, start + n):
        th = ph0 + k * cfg.step_m / rho
        eye = np.array([X / 2 + a * np.cos(th), Y / 2 + b * np.sin(th),
                        1.4 + 0.05 * np.sin(0.37 * k * cfg.step_m / rho * 7)])
        look = th + np.pi + 0.6 * np.sin(0.21 * th * 3) + 0.9
        tgt = np.array([X / 2 + 0.45 * X * np.cos(look), Y / 2 + 0.45 * Y * np.sin(look),
                        1.0 + 0.3 * np.sin(0.5 * th)])
        poses.append(look_pose(eye, tgt))
    return poses


# ----------------------------------------------------------------------------------------------
# frames
# ----------------------------------------------------------------------------------------------


def pixel_rays(cfg: SynthConfig, device="cpu"):
    """unit camera-frame ray directions for every pixel centre (row-major), float64."""
    v, u = torch.meshgrid(torch.arange(cfg.height, dtype=torch.float64, device=device),
                          torch.arange(cfg.width, dtype=torch.float64, device=device), indexing="ij")
    dc = torch.stack([(u - cfg.cx) / cfg.fx, (v - cfg.cy) / cfg.fy, torch.ones_like(u)], dim=-1)
    return dc.reshape(-1, 3)


@dataclass
class Frame:
    depth: torch.Tensor       # u16 [H,W] (raw sensor units)
    rgba: torch.Tensor        # u8  [H,W,4]
    R: np.ndarray             # f32 [3,3] camera->world
    t: np.ndarray             # f32 [3]
    depth_m: torch.Tensor     # f32 [H,W] exact analytic camera z (0 = no surface)
    rgb: torch.Tensor         # f32 [H,W,3] noise-free shaded colour
    normal: torch.Tensor      # f32 [H,W,3] world normals at the hits
    points: torch.Tensor      # f32 [H,W,3] world hit points


def render_frame(cfg: SynthConfig, scene: Scene, R, t, k: int = 0, device="cpu", dc=None) -> Frame:
    H, W = cfg.height, cfg.width
    if dc is None:
        dc = pixel_rays(cfg, device)
    Rt = torch.as_tensor(R, dtype=torch.float64, device=device)
    o = torch.as_tensor(t, dtype=torch.float64, device=device)
    dn = dc / dc.norm(dim=1, keepdim=True)
    dw = dn @ Rt.T
    tt, nrm, alb, valid, pts = scene.trace(o, dw)
    z = torch.where(valid, tt * dn[:, 2], torch.zeros_like(tt))
    exposure = 1.0
    if cfg.noise == "tof":
        exposure = float(1.0 + 0.03 * math.sin(0.7 * k))
    rgb = scene.shade(alb, nrm, dw, exposure)
    gen = torch.Generator(device=device)
    gen.manual_seed(cfg.seed * 100003 + k)
    zn = z.clone()
    keep = valid & (z >= cfg.range_min) & (z <= cfg.range_max)
    if cfg.noise == "kinect1":
        zn = zn + 1.5e-3 * zn * zn * torch.randn(zn.shape, generator=gen, device=device, dtype=zn.dtype)
    elif cfg.noise == "tof":
        zn = zn + (1.5e-3 + 2.5e-3 * zn) * torch.randn(zn.shape, generator=gen, device=device, dtype=zn.dtype)
    if cfg.dropout > 0:
        keep = keep & (torch.rand(zn.shape, generator=gen, device=device, dtype=zn.dtype) >= cfg.dropout)
        # grazing-angle dropouts (edges), like real sensors
        cosang = (nrm * dw).sum(dim=1).abs()
        keep = keep & (cosang > 0.12)
    raw = torch.round(zn * cfg.depth_scale).clamp(0, 65535)
    raw = torch.where(keep, raw, torch.zeros_like(raw))
    depth_u16 = raw.to(torch.int32).to(torch.uint16)
    rgb8 = torch.round(rgb * 255.0).clamp(0, 255).to(torch.uint8)
    rgba = torch.cat([rgb8, torch.full_like(rgb8[:, :1], 255)], dim=1)
    return Frame(depth=depth_u16.reshape(H, W), rgba=rgba.reshape(H, W, 4),
                 R=np.asarray(R, np.float32), t=np.asarray(t, np.float32),
                 depth_m=z.to(torch.float32).reshape(H, W), rgb=rgb.to(torch.float32).reshape(H, W, 3),
                 normal=nrm.to(torch.float32).reshape(H, W, 3), points=pts.to(torch.float32).reshape(H, W, 3))


def make_frames(cfg: SynthConfig, n: int, start: int = 0, device="cpu", scene: Scene | None = None):
    scene = scene or make_scene(cfg)
    dc = pixel_rays(cfg, device)
    return [render_frame(cfg, scene, R, t, start + i, device, dc)
            for i, (R, t) in enumerate(trajectory(cfg, n, start))]


def target_rgba(cfg: SynthConfig, frame: Frame) -> torch.Tensor:
    """Refinement target C_k.  cfg1 adds a 1-px stripe pattern that 5 mm voxels cannot hold,
    so the Gaussians receive a non-trivial gradient."""
    if cfg.scene != "plane_sphere":
        return frame.rgba
    rgba = frame.rgba.clone()
    u = torch.arange(cfg.width, device=rgba.device)
    stripe = ((u % 2) == 0)[None, :, None]
    rgb = rgba[..., :3].to(torch.int16)
    rgb = torch.where(stripe, (rgb + 40).clamp(max=255), (rgb - 40).clamp(min=0))
    rgba[..., :3] = rgb.to(torch.uint8)
    return rgba


# ----------------------------------------------------------------------------------------------
# Gaussians (input parameters; NOT the paper's adding rule, which is out of scope)
# ----------------------------------------------------------------------------------------------

_SH0_BASIS = 0.28209479177387814   # Y_00; used only to turn an albedo into a plausible sh0


def _quat_z_to(nrm: np.ndarray) -> np.ndarray:
    """quaternions (w,x,y,z) rotating local +z onto each unit normal."""
    z = np.array([0.0, 0.0, 1.0])
    out = np.zeros((nrm.shape[0], 4))
    c = nrm @ z
    ax = np.cross(np.broadcast_to(z, nrm.shape), nrm)
    s = np.linalg.norm(ax, axis=1)
    ang = np.arctan2(s, c)
    ax = np.where(s[:, None] > 1e-9, ax / np.maximum(s, 1e-12)[:, None], np.array([1.0, 0, 0]))
    out[:, 0] = np.cos(ang / 2)
    out[:, 1:] = ax * np.sin(ang / 2)[:, None]
    return out


def make_gaussians(cfg: SynthConfig, n: int | None = None, frames=None, seed: int | None = None,
                   sh_degree: int | None = None, n_view_frames: int = 8) -> dict:
    """N Gaussians on visible surfaces: random valid pixels of a few sequence frames are traced
    back to the analytic surface, offset +-2 mm along the normal; in-plane scales log-uniform in
    cfg.scale_mm, third scale 0.1x (disc, shortest axis on the normal); opacity U(0.1, 0.9);
    sh0 from the albedo-shaded colour + N(0, 0.1); other SH N(0, 0.02).  float32 numpy SoA."""
    n = cfg.n_gaussians if n is None else n
    deg = cfg.sh_degree if sh_degree is None else sh_degree
    rng = np.random.default_rng(5000 + (cfg.seed if seed is None else seed))
    if frames is None:
        span = max(1, min(cfg.n_frames, 600))
        idx = sorted({int(i) for i in np.linspace(0, span - 1, n_view_frames)})
        scene = make_scene(cfg)
        poses = trajectory(cfg, span)
        frames = [render_frame(cfg, scene, *poses[i], k=i) for i in idx]
    pts_all, nrm_all, col_all = [], [], []
    per = -(-n // len(frames))
    for f in frames:
        valid = (f.depth_m.reshape(-1) > 0.0).numpy()
        ids = np.nonzero(valid)[0]
        pick = rng.choice(ids, size=per, replace=True)
        pts_all.append(f.points.reshape(-1, 3).numpy()[pick])
        nrm_all.append(f.normal.reshape(-1, 3).numpy()[pick])
        col_all.append(f.rgb.reshape(-1, 3).numpy()[pick])
    pts = np.concatenate(pts_all)[:n].astype(np.float64)
    nrm = np.concatenate(nrm_all)[:n].astype(np.float64)
    col = np.concatenate(col_all)[:n].astype(np.float64)
    nrm /= np.maximum(np.linalg.norm(nrm, axis=1, keepdims=True), 1e-12)
    xyz = pts + nrm * rng.uniform(-0.002, 0.002, size=(n, 1))
    lo, hi = cfg.scale_mm
    s1 = np.exp(rng.uniform(np.log(lo * 1e-3), np.log(hi * 1e-3), size=n))
    log_scale = np.log(np.stack([s1, s1, 0.1 * s1], axis=1))
    rot = _quat_z_to(nrm)
    # random in-plane spin and a non-unit norm (the forward pass normalises)
    spin = rng.uniform(0, 2 * np.pi, size=n)
    qs = np.stack([np.cos(spin / 2), np.zeros(n), np.zeros(n), np.sin(spin / 2)], axis=1)
    rot = _qmul(rot, qs) * rng.uniform(0.7, 1.4, size=(n, 1))
    sig = rng.uniform(0.1, 0.9, size=n)
    op = np.log(sig / (1 - sig))
    nc = (deg + 1) ** 2
    sh = rng.normal(0.0, 0.02, size=(n, nc, 3))
    sh[:, 0, :] = (col - 0.5) / _SH0_BASIS + rng.normal(0, 0.1, size=(n, 3))
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return {"sh_degree": deg, "xyz": f32(xyz), "log_scale": f32(log_scale), "rot": f32(rot),
            "opacity_raw": f32(op), "sh": f32(sh.reshape(n, nc * 3))}


def _qmul(a, b):
    w1, x1, y1, z1 = a.T
    w2, x2, y2, z2 = b.T
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], axis=1)


def random_gaussians(n: int, deg: int, rng: np.random.Generator, center=(0.0, 0.0, 1.0),
                     spread=0.1, scale=(0.005, 0.05)) -> dict:
    """Small random scenes for gradient / binning tests (free position, anisotropic scale)."""
    c = np.asarray(center)
    xyz = c + rng.uniform(-spread, spread, size=(n, 3))
    ls = np.log(rng.uniform(scale[0], scale[1], size=(n, 3)))
    rot = rng.normal(size=(n, 4))
    op = rng.normal(0.0, 1.0, size=n)
    nc = (deg + 1) ** 2
    sh = rng.normal(0.0, 0.3, size=(n, nc * 3))
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return {"sh_degree": deg, "xyz": f32(xyz), "log_scale": f32(ls), "rot": f32(rot),
            "opacity_raw": f32(op), "sh": f32(sh)}


def sdf_stage_inputs(cfg: SynthConfig, frame: Frame, seed: int = 0, miss_frac: float = 0.02):
    """Seeded stand-ins for a raycast's (D_t, C_t) so the render stage can be tested at full
    size without consuming any CUDA output: D_t = exact analytic depth with a few misses,
    C_t = the shaded colour blurred and perturbed (the SDF's smoother colour)."""
    rng = np.random.default_rng(7000 + seed)
    Dt = frame.depth_m.numpy().astype(np.float32).copy()
    miss = rng.random(Dt.shape) < miss_frac
    Dt[miss] = 0.0
    rgb = frame.rgb.numpy().astype(np.float64)
    k = np.array([0.25, 0.5, 0.25])
    blur = rgb.copy()
    blur[1:-1] = k[0] * rgb[:-2] + k[1] * rgb[1:-1] + k[2] * rgb[2:]
    blur[:, 1:-1] = k[0] * blur[:, :-2] + k[1] * blur[:, 1:-1] + k[2] * blur[:, 2:]
    Ct = np.clip(blur + rng.normal(0, 0.02, size=blur.shape), 0, 1).astype(np.float32)
    Ct[Dt == 0] = 0.0
    return Dt, Ct


def adding_stage_inputs(cfg: SynthConfig, frame: Frame, seed: int = 0, miss_frac: float = 0.02):
    """Seeded stand-ins for the inputs of Gaussian adding, so adding can be
    tested without consuming any CUDA output: V* = the analytic hit points (a raycast vertex map),
    D_t = their camera depth with a few misses, C* = the shaded colour perturbed by N(0, 0.04)
    (a render whose error exceeds delta_c on part of the image), W_G ~ U(0, 8), target C_k =
    the frame's colour.  No arithmetic of the method: only the scene, noise and masks."""
    rng = np.random.default_rng(9000 + seed)
    Dt = frame.depth_m.numpy().astype(np.float32).copy()
    Dt[rng.random(Dt.shape) < miss_frac] = 0.0
    V = frame.points.numpy().astype(np.float32).copy()
    V[Dt == 0] = 0.0
    rgb = frame.rgb.numpy().astype(np.float64)
    Cs = np.clip(rgb + rng.normal(0, 0.04, size=rgb.shape), 0, 1).astype(np.float32)
    WG = rng.uniform(0, 8, size=Dt.shape).astype(np.float32)
    return {"V": V, "Dt": Dt, "Cstar": Cs, "WG": WG, "target": frame.rgba.numpy()}
