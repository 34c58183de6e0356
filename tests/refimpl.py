"""Test-only independent torch-fp64 implementation of the render path (projection, Eqs. 1-4,
L1), written from PAPER.md and the DESIGN.md readings with a different structure from
oracle.c (matrix algebra, quaternion sandwich products, all-pairs over every pixel, torch
autograd for the gradient).  It pins the oracle: a dropped term, a wrong sign or index or a
transposed operand in either implementation makes them disagree.  Not part of libgps or the
oracle."""
from __future__ import annotations

import numpy as np
import torch

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = [1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
         0.5462742152960396]
SH_C3 = [-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
         -0.4570457994644658, 1.445305721320277, -0.5900435899266435]


def sh_eval(deg, sh, d):
    """sh: (n, nc, 3), d: (n, 3) unit -> (n, 3)."""
    x, y, z = d[:, 0:1], d[:, 1:2], d[:, 2:3]
    r = SH_C0 * sh[:, 0]
    if deg > 0:
        r = r - SH_C1 * y * sh[:, 1] + SH_C1 * z * sh[:, 2] - SH_C1 * x * sh[:, 3]
    if deg > 1:
        xx, yy, zz, xy, yz, xz = x * x, y * y, z * z, x * y, y * z, x * z
        r = (r + SH_C2[0] * xy * sh[:, 4] + SH_C2[1] * yz * sh[:, 5]
             + SH_C2[2] * (2 * zz - xx - yy) * sh[:, 6] + SH_C2[3] * xz * sh[:, 7]
             + SH_C2[4] * (xx - yy) * sh[:, 8])
    if deg > 2:
        r = (r + SH_C3[0] * y * (3 * xx - yy) * sh[:, 9] + SH_C3[1] * xy * z * sh[:, 10]
             + SH_C3[2] * y * (4 * zz - xx - yy) * sh[:, 11]
             + SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy) * sh[:, 12]
             + SH_C3[4] * x * (4 * zz - xx - yy) * sh[:, 13]
             + SH_C3[5] * z * (xx - yy) * sh[:, 14] + SH_C3[6] * x * (xx - 3 * yy) * sh[:, 15])
    return r


def quat_rotmat(q):
    """R(q) for unit q=(w,x,y,z), built by rotating the basis vectors with q v q*."""
    w, v = q[:, :1], q[:, 1:]
    cols = []
    for k in range(3):
        e = torch.zeros_like(v)
        e[:, k] = 1.0
        # q e q* = e + 2w (v x e) + 2 v x (v x e)
        c1 = torch.cross(v, e, dim=1)
        cols.append(e + 2 * w * c1 + 2 * torch.cross(v, c1, dim=1))
    return torch.stack(cols, dim=2)  # column k = R e_k


F32 = lambda x: float(np.float32(x))  # the config constants as the fp32 values both sides see


def project(params, cam, R, t, near_z=F32(0.2), lowpass=F32(0.3)):
    """params: dict of torch fp64 tensors (xyz, log_scale, rot, opacity_raw, sh (n,nc,3)).
    Returns dict with p_hat (n,2), conic (n,2,2), depth, sigma, color, valid mask."""
    fx, fy, cx, cy, W, H = cam
    Rw = torch.as_tensor(R, dtype=torch.float64).reshape(3, 3)
    tw = torch.as_tensor(t, dtype=torch.float64).reshape(3)
    p = params["xyz"]
    X = (p - tw) @ Rw  # rows: R^T (p - t)
    z = X[:, 2]
    s = torch.exp(params["log_scale"])
    q = params["rot"] / params["rot"].norm(dim=1, keepdim=True)
    Rq = quat_rotmat(q)
    M = Rq * s[:, None, :]
    Sig = M @ M.transpose(1, 2)
    limx = 1.3 * (W / (2 * fx))
    limy = 1.3 * (H / (2 * fy))
    u = torch.clamp(X[:, 0] / z, -limx, limx)
    v = torch.clamp(X[:, 1] / z, -limy, limy)
    n = p.shape[0]
    J = torch.zeros(n, 2, 3, dtype=torch.float64)
    J[:, 0, 0] = fx / z
    J[:, 0, 2] = -fx * u / z
    J[:, 1, 1] = fy / z
    J[:, 1, 2] = -fy * v / z
    T = J @ Rw.T  # J * (world->camera rotation)
    S2 = T @ Sig @ T.transpose(1, 2) + lowpass * torch.eye(2, dtype=torch.float64)
    conic = torch.linalg.inv(S2)
    ph = torch.stack([fx * X[:, 0] / z + cx, fy * X[:, 1] / z + cy], dim=1)
    sigma = torch.sigmoid(params["opacity_raw"])
    dvec = p - tw
    d = dvec / dvec.norm(dim=1, keepdim=True)
    deg = int(round(params["sh"].shape[1] ** 0.5)) - 1
    col = torch.clamp_min(sh_eval(deg, params["sh"], d) + 0.5, 0.0)
    valid = (z > near_z) & (torch.linalg.det(S2) > 0)
    return {"p_hat": ph, "conic": conic, "S2": S2, "depth": z, "sigma": sigma, "color": col,
            "valid": valid}


def render_allpairs(params, cam, R, t, Dt, Ct, eps=F32(0.02), alpha_min=F32(1 / 255),
                    near_z=F32(0.2), lowpass=F32(0.3)):
    """Eqs. 1-4 over ALL (Gaussian, pixel) pairs, indicators computed without gradient."""
    fx, fy, cx, cy, W, H = cam
    pr = project(params, cam, R, t, near_z, lowpass)
    ys, xs = torch.meshgrid(torch.arange(H, dtype=torch.float64), torch.arange(W, dtype=torch.float64),
                            indexing="ij")
    pix = torch.stack([xs.reshape(-1), ys.reshape(-1)], dim=1)  # (P,2)
    delta = pix[None, :, :] - pr["p_hat"][:, None, :]  # (n,P,2)
    qf = torch.einsum("npi,nij,npj->np", delta, pr["conic"], delta)
    alpha = pr["sigma"][:, None] * torch.exp(-0.5 * qf)
    Dt_t = torch.as_tensor(np.asarray(Dt, np.float64).reshape(-1))
    with torch.no_grad():
        ind = (pr["valid"][:, None] & (qf <= 9.0) & (alpha >= alpha_min)
               & ((Dt_t[None, :] == 0) | (pr["depth"][:, None] < Dt_t[None, :] + eps)))
    a = torch.where(ind, alpha, torch.zeros_like(alpha))
    CG = a.T @ pr["color"]  # (P,3)
    WG = a.sum(dim=0)
    Ct_t = torch.as_tensor(np.asarray(Ct, np.float64).reshape(-1, 3))
    Cs = (Ct_t + CG) / (1.0 + WG)[:, None]
    return Cs.reshape(H, W, 3), WG.reshape(H, W), ind


def to_torch_params(g, requires_grad=False):
    n = g["xyz"].shape[0]
    nc = (int(g["sh_degree"]) + 1) ** 2
    out = {
        "xyz": torch.tensor(np.asarray(g["xyz"], np.float64)),
        "log_scale": torch.tensor(np.asarray(g["log_scale"], np.float64)),
        "rot": torch.tensor(np.asarray(g["rot"], np.float64)),
        "opacity_raw": torch.tensor(np.asarray(g["opacity_raw"], np.float64).reshape(n)),
        "sh": torch.tensor(np.asarray(g["sh"], np.float64).reshape(n, nc, 3)),
    }
    if requires_grad:
        for v in out.values():
            v.requires_grad_(True)
    return out


def rot_z(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]])


def rot_x(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[1.0, 0, 0], [0, c, -s], [0, s, c]])


def rot_y(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, 0, s], [0, 1.0, 0], [-s, 0, c]])


def random_rotation(rng):
    return (rot_z(rng.uniform(-np.pi, np.pi)) @ rot_x(rng.uniform(-0.5, 0.5))
            @ rot_y(rng.uniform(-0.5, 0.5))).astype(np.float32)
