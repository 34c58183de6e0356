"""CPU oracle of Gaussian adding and removal -- TEST INFRASTRUCTURE ONLY.

Plain numpy, one definition per function, in the paper's order:

* :func:`vertex_normals`  -- N*_k from the raycast vertex map V*_k ("raycast vertex map and
                             normal map"; reading R-NORMAL).
* :func:`add_mask`        -- Eq. 6: |C* - C_k| > delta_c and W_G < delta_W (R-ADD-MASK).
* :func:`sample_keep`     -- "uniformly sample 25% pixels on M", as a counter-based hash
                             both sides implement (R-SAMPLE).
* :func:`knn_scale`       -- App. A: s1 from the 3 vertices of M nearest to V*(u),
                             truncated at 0.1 (R-KNN: the garbled sqrt(1/3 sum ||.||) read as RMS).
* :func:`init_gaussians`  -- P:124: p = V*(u), SH0 from C_k(u), disc with its shortest axis on
                             N*(u), opacity 0.5 (R-INIT).
* :func:`remove_mask`     -- Eq. 8: sigma < 0.005 or max s > 0.1 or max s < 0.003
                             (R-REMOVE), decided on the raw parameters against fp32 thresholds.

Decisions that produce integers (mask, sample, removal) are taken in fp32 with the same rounding
the CUDA path uses; continuous values are fp64.  Nothing here imports or
consumes the CUDA path.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial import cKDTree

C0 = 0.28209479177387814  # SH degree-0 basis constant (3DGS)


def vertex_normals(V: np.ndarray, D: np.ndarray, cam_t) -> np.ndarray:
    """R-NORMAL: N(u,v) = normalise((V(u+1,v) - V(u-1,v)) x (V(u,v+1) - V(u,v-1))), turned to face
    the camera centre; zero where the pixel or any of the four neighbours has no hit (D = 0) or
    lies on the image border, or the cross product vanishes.  V, N: [H, W, 3] world, fp64."""
    V = np.asarray(V, np.float64)
    H, W, _ = V.shape
    N = np.zeros((H, W, 3))
    ok = np.zeros((H, W), bool)
    hit = np.asarray(D) > 0
    ok[1:-1, 1:-1] = hit[1:-1, 1:-1] & hit[1:-1, 2:] & hit[1:-1, :-2] & hit[2:, 1:-1] & hit[:-2, 1:-1]
    dx = V[1:-1, 2:] - V[1:-1, :-2]
    dy = V[2:, 1:-1] - V[:-2, 1:-1]
    n = np.cross(dx, dy)
    nn = np.linalg.norm(n, axis=-1)
    inner = ok[1:-1, 1:-1] & (nn > 0)
    n = np.where(inner[..., None], n / np.where(nn > 0, nn, 1.0)[..., None], 0.0)
    away = np.einsum("ijk,ijk->ij", n, V[1:-1, 1:-1] - np.asarray(cam_t, np.float64)) > 0
    n = np.where(away[..., None], -n, n)
    N[1:-1, 1:-1] = n
    return N


def add_mask(Cstar, WG, Dt, N, target_rgba, delta_c=0.05, delta_w=4.0) -> np.ndarray:
    """R-ADD-MASK (Eq. 6): pixel u is in M iff it has an SDF hit and a normal (V*, N* defined),
    max_ch |C*_ch - C_k,ch| > delta_c and W_G < delta_W.  Evaluated in fp32: C_k = c8 * fl(1/255),
    d = |C* - C_k| (one rounding each), compared with fl(delta_c); W_G with fl(delta_W)."""
    f = np.float32
    ck = np.asarray(target_rgba)[..., :3].astype(f) * f(1.0 / 255.0)
    d = np.abs(np.asarray(Cstar, f) - ck)
    big = (d > f(delta_c)).any(axis=-1)
    valid = (np.asarray(Dt) > 0) & (np.abs(np.asarray(N)).sum(axis=-1) > 0)
    return valid & big & (np.asarray(WG, f) < f(delta_w))


def hash32(x: np.ndarray) -> np.ndarray:
    """lowbias32 integer mixer (uint32 -> uint32)."""
    x = np.asarray(x, np.uint32).copy()
    x ^= x >> np.uint32(16)
    x *= np.uint32(0x7FEB352D)
    x ^= x >> np.uint32(15)
    x *= np.uint32(0x846CA68B)
    x ^= x >> np.uint32(16)
    return x


def sample_keep(n_pixels: int, seed: int, frac: float = 0.25) -> np.ndarray:
    """R-SAMPLE: pixel index i is sampled iff hash32(i ^ hash32(seed)) < floor(frac * 2^32)."""
    thr = np.uint64(int(frac * 4294967296.0))
    h = hash32(np.arange(n_pixels, dtype=np.uint32) ^ hash32(np.array([seed], np.uint32))[0])
    return h.astype(np.uint64) < thr


def knn_scale(Vm: np.ndarray, q_idx: np.ndarray, s_max: float = 0.1):
    """R-KNN (App. A): for each query q (an index into the mask vertices Vm [M, 3]), the 3 other
    vertices of M nearest to Vm[q] (Euclidean, fp64), s1 = min(s_max, sqrt((d1^2+d2^2+d3^2)/3));
    fewer than 3 other vertices -> s_max.  Returns (s1, tie) where tie flags queries whose 3rd and
    4th distances agree to 1e-5 relative (the neighbour set is then ambiguous in fp32)."""
    Vm = np.asarray(Vm, np.float64)
    q_idx = np.asarray(q_idx, np.int64)
    s = np.full(len(q_idx), float(s_max))
    tie = np.zeros(len(q_idx), bool)
    if len(Vm) < 4 or len(q_idx) == 0:
        return s, tie
    k = min(5, len(Vm))
    dist, idx = cKDTree(Vm).query(Vm[q_idx], k=k)
    # drop the query itself (distance 0 at its own index); duplicates of its position stay
    own = idx == q_idx[:, None]
    d = np.where(own, np.inf, dist)
    d.sort(axis=1)
    d3 = d[:, :3]
    rms = np.sqrt((d3 ** 2).sum(axis=1) / 3.0)
    s = np.minimum(rms, s_max)
    if d.shape[1] >= 4:
        tie = np.abs(d[:, 3] - d[:, 2]) <= 1e-5 * np.maximum(d[:, 2], 1e-12)
    return s, tie


def quat_z_to(n: np.ndarray) -> np.ndarray:
    """Unit quaternion (w, x, y, z) of the shortest rotation taking e_z to the unit vector n
    (for n = -e_z: the half-turn about e_x)."""
    n = np.asarray(n, np.float64)
    w = 1.0 + n[..., 2]
    q = np.stack([w, -n[..., 1], n[..., 0], np.zeros_like(w)], -1)
    flip = w <= 1e-12
    q[flip] = np.array([0.0, 1.0, 0.0, 0.0])
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def init_gaussians(V, N, target_rgba, sel: np.ndarray, s1: np.ndarray, sh_degree: int, opacity=0.5) -> dict:
    """R-INIT (App. A): one Gaussian per selected pixel (row-major pixel order):
    p = V*(u); SH0 = (C_k(u) - 0.5) / C0 so that the degree-0 colour is C_k(u), higher SH 0;
    opacity_raw = logit(opacity); rotation taking e_z to N*(u) (shortest axis on the normal);
    scales (s1, s1, 0.1 s1) stored as logs."""
    H, W = np.asarray(V).shape[:2]
    ii = np.flatnonzero(sel.reshape(-1))
    Vf = np.asarray(V, np.float64).reshape(-1, 3)[ii]
    Nf = np.asarray(N, np.float64).reshape(-1, 3)[ii]
    ck = np.asarray(target_rgba).reshape(-1, 4)[ii, :3].astype(np.float64) / 255.0
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((len(ii), nc * 3))
    sh[:, :3] = (ck - 0.5) / C0
    ls = np.log(np.stack([s1, s1, 0.1 * s1], -1))
    return {"xyz": Vf, "log_scale": ls, "rot": quat_z_to(Nf),
            "opacity_raw": np.full(len(ii), np.log(opacity / (1.0 - opacity))), "sh": sh,
            "sh_degree": sh_degree, "pixels": ii}


def remove_thresholds(sigma_min=0.005, s_max=0.1, s_min=0.003):
    """fp32 thresholds on the raw parameters, each rounded once from double: sigmoid(o) < sigma_min
    iff o < logit(sigma_min); max exp(ls) > s_max iff max ls > ln s_max (likewise s_min)."""
    f = np.float32
    return f(np.log(sigma_min / (1.0 - sigma_min))), f(np.log(s_max)), f(np.log(s_min))


def remove_mask(opacity_raw, log_scale, sigma_min=0.005, s_max=0.1, s_min=0.003) -> np.ndarray:
    """R-REMOVE (Eq. 8): True = delete.  Decided in fp32 on the raw parameters."""
    to, tmax, tmin = remove_thresholds(sigma_min, s_max, s_min)
    o = np.asarray(opacity_raw, np.float32)
    mx = np.asarray(log_scale, np.float32).max(axis=-1)
    return (o < to) | (mx > tmax) | (mx < tmin)


def compact(arrays: dict, keep: np.ndarray) -> dict:
    """Stable removal: survivors keep their relative order (every per-Gaussian array alike)."""
    return {k: (np.asarray(v)[keep] if isinstance(v, np.ndarray) and v.ndim >= 1 and len(v) == len(keep) else v)
            for k, v in arrays.items()}
