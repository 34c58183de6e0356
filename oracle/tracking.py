"""CPU oracle of the ICP camera tracking of Eq. 5 -- TEST INFRASTRUCTURE ONLY.

PAPER.md P:108-113: "We adopt the standard ICP method for camera tracking ... which minimizes the
point-to-plane distance E(xi) = sum |(T_gk V_k^l(u) - V*_{k-1}(u^)) . N*_{k-1}(u^)| ... A
resolution hierarchy of the depth map is used".  The projection u^ = pi(K T_{g,k-1} V_k^l(u)) is
garbled (no inverse, no composition with T_gk); reading R-ICP-ASSOC:
u^ = pi(K T_{g,k-1}^{-1} T_gk V_k^l(u)), the current estimate's point projected into the camera the
model maps were raycast from.  Readings R-ICP-*: DESIGN.md §3.

Plain numpy fp64, step by step: depth pyramid -> vertex / normal maps -> per level, per
iteration: projective association, gates, linearised point-to-plane system (Gauss-Newton on a
left-multiplied twist), solve, pose update.  Shares nothing with the CUDA path.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class IcpCfg:
    levels: int = 3
    iters: tuple = (10, 5, 4)       # finest -> coarsest (SPEC: 4, 5, 10 coarse -> fine)
    dist_max: float = 0.1           # metres (SPEC gate)
    angle_max_deg: float = 30.0     # SPEC gate
    depth_min: float = 0.1
    depth_max: float = 10.0
    eps: float = 1e-6               # convergence on |xi|
    min_inlier_frac: float = 0.1
    min_inlier_px_frac: float = 0.05  # R-ICP-FAIL: and inliers >= this fraction of the frame's pixels
    min_pivot_ratio: float = 1e-3     # R-ICP-FAIL: and the last system's smallest Cholesky pivot /
                                      # largest diagonal >= this
    filter_radius: int = 0            # R-ICP-FILT: bilateral pre-filter radius (0 = off)
    filter_sigma_s: float = 4.5
    filter_sigma_r: float = 0.03


def bilateral(d: np.ndarray, r: int, sigma_s: float, sigma_r: float) -> np.ndarray:
    """R-ICP-FILT (KinectFusion's measurement filter), written out: for every valid pixel (d > 0),
    sum_q w_q d_q / sum_q w_q over the valid pixels q of the (2r+1)^2 window inside the image,
    w_q = exp(-|q - p|^2 / (2 sigma_s^2) - (d_q - d_p)^2 / (2 sigma_r^2)); invalid pixels stay 0."""
    d = np.asarray(d, np.float64)
    H, W = d.shape
    sw = np.zeros_like(d)
    sz = np.zeros_like(d)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            q = np.zeros_like(d)  # d shifted so that q[y, x] = d[y + dy, x + dx] (0 outside)
            ys, yd = slice(max(dy, 0), H + min(dy, 0)), slice(max(-dy, 0), H + min(-dy, 0))
            xs, xd = slice(max(dx, 0), W + min(dx, 0)), slice(max(-dx, 0), W + min(-dx, 0))
            q[yd, xd] = d[ys, xs]
            w = np.exp(-(dx * dx + dy * dy) / (2 * sigma_s ** 2) - (q - d) ** 2 / (2 * sigma_r ** 2)) * (q > 0)
            sw += w
            sz += w * q
    return np.where(d > 0, sz / np.maximum(sw, 1e-300), 0.0)


def depth_pyramid(depth_m: np.ndarray, levels: int, dmin: float, dmax: float):
    """R-ICP-PYR: level 0 = depth in metres, invalid (0) outside [dmin, dmax]; level l+1 at (u,v) =
    mean of the valid depths among the 2x2 children (2u..2u+1, 2v..2v+1), 0 if none is valid."""
    d = np.asarray(depth_m, np.float64).copy()
    d[(d < dmin) | (d > dmax)] = 0.0
    out = [d]
    for _ in range(1, levels):
        p = out[-1]
        H, W = p.shape[0] // 2, p.shape[1] // 2
        c = p[:2 * H, :2 * W].reshape(H, 2, W, 2)
        n = (c > 0).sum(axis=(1, 3))
        s = c.sum(axis=(1, 3))
        out.append(np.where(n > 0, s / np.maximum(n, 1), 0.0))
    return out


def level_intrinsics(fx, fy, cx, cy, level):
    """Intrinsics of pyramid level l (pixel centres at integer coordinates): f / 2^l and
    c' = (c + 0.5) / 2^l - 0.5."""
    s = 2.0 ** level
    return fx / s, fy / s, (cx + 0.5) / s - 0.5, (cy + 0.5) / s - 0.5


def backproject(d: np.ndarray, fx, fy, cx, cy):
    H, W = d.shape
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    return np.stack([(u - cx) / fx * d, (v - cy) / fy * d, d], -1)


def normals(V: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """R-NORMAL on a vertex map in camera coordinates (the camera at the origin)."""
    H, W, _ = V.shape
    N = np.zeros((H, W, 3))
    ok = np.zeros((H, W), bool)
    ok[1:-1, 1:-1] = valid[1:-1, 1:-1] & valid[1:-1, 2:] & valid[1:-1, :-2] & valid[2:, 1:-1] & valid[:-2, 1:-1]
    n = np.cross(V[1:-1, 2:] - V[1:-1, :-2], V[2:, 1:-1] - V[:-2, 1:-1])
    nn = np.linalg.norm(n, axis=-1)
    inner = ok[1:-1, 1:-1] & (nn > 0)
    n = np.where(inner[..., None], n / np.where(nn > 0, nn, 1)[..., None], 0.0)
    flip = np.einsum("ijk,ijk->ij", n, V[1:-1, 1:-1]) > 0
    N[1:-1, 1:-1] = np.where(flip[..., None], -n, n)
    return N


def subsample(M: np.ndarray, level: int) -> np.ndarray:
    """Model maps of level l: every 2^l-th pixel of the full-resolution raycast maps."""
    s = 2 ** level
    return M[::s, ::s][: M.shape[0] // s, : M.shape[1] // s]


def skew(w):
    return np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])


def exp_se3(xi):
    """Left-multiplied increment of the twist xi = (v, w): rotation by Rodrigues, translation v
    (p' = R_w p + v, the first-order form p + v + w x p)."""
    v, w = np.asarray(xi[:3], np.float64), np.asarray(xi[3:], np.float64)
    th = np.linalg.norm(w)
    K = skew(w)
    if th < 1e-12:
        R = np.eye(3) + K
    else:
        R = np.eye(3) + np.sin(th) / th * K + (1 - np.cos(th)) / th ** 2 * K @ K
    return R, v


def system(Vc, Nc, R, t, Vm, Nm, Rp, tp, intr, cfg: IcpCfg):
    """The linearised Eq. 5 over the inliers of one level: A = sum J^T J, b = sum J r, E = sum r^2,
    count.  Current point p = R Vc + t (world), normal n = R Nc; u^ = nearest pixel of p in the
    previous camera (R-ICP-ASSOC); q = Vm(u^), m = Nm(u^); gates |p - q| < dist_max and
    n . m > cos(angle_max) (R-ICP-GATE); r = (p - q) . m; J = [m, p x m]."""
    fx, fy, cx, cy = intr
    H, W = Vm.shape[:2]
    ok = np.abs(Nc).sum(-1) > 0
    p = Vc[ok] @ R.T + t
    n = Nc[ok] @ R.T
    x = (p - tp) @ Rp                       # previous camera coordinates: Rp^T (p - tp)
    z = x[:, 2]
    front = z > 1e-9
    u = np.floor(fx * x[:, 0] / np.where(front, z, 1) + cx + 0.5)
    v = np.floor(fy * x[:, 1] / np.where(front, z, 1) + cy + 0.5)
    inb = front & (u >= 0) & (u <= W - 1) & (v >= 0) & (v <= H - 1)
    ui, vi = u[inb].astype(int), v[inb].astype(int)
    q, m = Vm[vi, ui], Nm[vi, ui]
    p, n = p[inb], n[inb]
    has = np.abs(m).sum(-1) > 0
    d = p - q
    keep = has & (np.linalg.norm(d, axis=-1) < cfg.dist_max) & ((n * m).sum(-1) > np.cos(np.radians(cfg.angle_max_deg)))
    p, m, d = p[keep], m[keep], d[keep]
    r = (d * m).sum(-1)
    J = np.concatenate([m, np.cross(p, m)], 1)
    return J.T @ J, J.T @ r, float((r * r).sum()), int(keep.sum()), int(ok.sum())


def track(depth_u16, depth_scale, K, Vm_full, Nm_full, Rp, tp, R0, t0, cfg: IcpCfg = IcpCfg()):
    """Frame-to-model ICP (Eq. 5): coarse -> fine over the pyramid, cfg.iters[l] Gauss-Newton
    steps at level l (stopping early when |xi| < eps).  Returns (R, t, info)."""
    fx, fy, cx, cy = K
    d = np.asarray(depth_u16, np.float64) * np.float64(np.float32(1.0 / depth_scale))
    if cfg.filter_radius > 0:  # R-ICP-FILT on the in-range level-0 depth, before the pyramid
        d0 = d.copy()
        d0[(d0 < cfg.depth_min) | (d0 > cfg.depth_max)] = 0.0
        d = bilateral(d0, cfg.filter_radius, cfg.filter_sigma_s, cfg.filter_sigma_r)
    pyr = depth_pyramid(d, cfg.levels, cfg.depth_min, cfg.depth_max)
    R, t = np.asarray(R0, np.float64).copy(), np.asarray(t0, np.float64).copy()
    Rp, tp = np.asarray(Rp, np.float64), np.asarray(tp, np.float64)
    info = {"steps": 0, "inliers": 0, "valid": 0, "degenerate": False, "pivot_ratio": 0.0}
    for lev in reversed(range(cfg.levels)):
        intr = level_intrinsics(fx, fy, cx, cy, lev)
        Vc = backproject(pyr[lev], *intr)
        Nc = normals(Vc, pyr[lev] > 0)
        Vm, Nm = subsample(np.asarray(Vm_full, np.float64), lev), subsample(np.asarray(Nm_full, np.float64), lev)
        for _ in range(cfg.iters[lev]):
            A, b, E, cnt, nval = system(Vc, Nc, R, t, Vm, Nm, Rp, tp, intr, cfg)
            info.update(inliers=cnt, valid=nval, energy=E)
            if cnt < 6:
                info["degenerate"] = True
                break
            ev = np.linalg.eigvalsh(A)
            if ev[0] <= 1e-12 * max(ev[-1], 1e-300):
                info["degenerate"] = True
                break
            Lc = np.linalg.cholesky(A)
            info["pivot_ratio"] = float((np.diag(Lc) ** 2).min() / np.diag(A).max())
            xi = -np.linalg.solve(A, b)
            dR, dt = exp_se3(xi)
            R, t = dR @ R, dR @ t + dt
            info["steps"] += 1
            if np.linalg.norm(xi) < cfg.eps:
                break
    info["inlier_frac"] = info["inliers"] / max(info["valid"], 1)
    info["converged"] = ((not info["degenerate"]) and info["inlier_frac"] >= cfg.min_inlier_frac
                         and info["inliers"] >= cfg.min_inlier_px_frac * np.shape(depth_u16)[0] * np.shape(depth_u16)[1]
                         and info["pivot_ratio"] >= cfg.min_pivot_ratio)
    return R, t, info
