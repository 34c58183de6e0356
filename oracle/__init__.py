"""CPU oracle for the GPS-SLAM mapping step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the CUDA path
(``paper_2509_11574_b200``) and never consumes anything that path produced.

The heavy loops are plain C in ``oracle.c`` (built by :func:`build`); this module adds the
numpy-fp64 pieces that are one formula each:

* :func:`l1_loss`       -- Eq. 7 with reading R-L1 (mean over the mask).
* :func:`adam_step`     -- torch's Adam formula ("Libtorch"), learning rates of App. C.
* :func:`tile_lists`    -- the (tile, depth, index)-ordered per-tile lists (plain definition,
                           DESIGN.md §4.3), via numpy's lexsort as the sort primitive.

Citations are PAPER.md lines (``P:n``); readings ``R-*`` are listed in DESIGN.md §3.
Parity pins live in ``tests/test_oracle_*.py``; nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fno-math-errno",
           "-shared", "-fPIC"]


_LIB_OMP_PATH = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -ffp-contract=off) and, for the CPU timing
    baseline only, liboracle_omp.so (the same source with -fopenmp: pixel, block, Gaussian and
    row-band loops in parallel; each pixel still sums in index order)."""
    for path, extra in ((_LIB_PATH, []), (_LIB_OMP_PATH, ["-fopenmp"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
            tmp = path + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", *_CFLAGS, *extra, _SRC, "-o", tmp, "-lm"])
            os.replace(tmp, path)
    return _LIB_PATH


_lib = None
_use_omp = False


def use_openmp(on: bool = True) -> int:
    """Switch this process to the OpenMP build (bench.py's cpu_baseline only; tests never call
    it).  Returns the number of threads it will use."""
    global _use_omp, _lib
    if on != _use_omp:
        _use_omp = on
        _lib = None
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)) if on else 1


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_OMP_PATH if _use_omp else _LIB_PATH)
        vp, i64, i32, f32, f64 = C.c_void_p, C.c_int64, C.c_int, C.c_float, C.c_double
        L.orc_volume_new.restype = vp
        L.orc_volume_new.argtypes = [f32, f32, i32, f32, f32, i64]
        L.orc_volume_free.argtypes = [vp]
        L.orc_volume_n.restype = i64
        L.orc_volume_n.argtypes = [vp]
        L.orc_volume_nvis.restype = i64
        L.orc_volume_nvis.argtypes = [vp]
        L.orc_volume_overflow.argtypes = [vp]
        L.orc_volume_export.argtypes = [vp, vp, vp, vp]
        L.orc_volume_export_visible.argtypes = [vp, vp]
        L.orc_fuse.argtypes = [vp, vp, i32, i32, vp, vp, vp, f32, vp]
        L.orc_raycast.argtypes = [vp, vp, i32, i32, vp, vp, vp, i64, vp, vp, vp, vp]
        L.orc_project_p32.argtypes = [i64, vp, vp, vp, vp, i32, i32, vp, vp, f32, f32, vp, vp, vp]
        L.orc_project_p32_full.argtypes = [i64, vp, vp, vp, vp, vp, i32, i32, vp, vp, f32, f32, vp, vp, vp, vp]
        L.orc_sh_basis.argtypes = [f64, f64, f64, vp, vp]
        L.orc_render.argtypes = [i64, i32, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp,
                                 f64, f64, f64, f64, vp, vp, vp, vp, vp, vp]
        L.orc_backward.argtypes = [i64, i32, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp,
                                   f64, f64, f64, f64, vp, vp, vp, vp, vp,
                                   vp, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ----------------------------------------------------------------------------------------------
# Camera helpers (reading R-PIX / R-POSE): intrinsics (fx, fy, cx, cy, W, H), pose R (3x3 row
# major, camera->world) and t.
# ----------------------------------------------------------------------------------------------
@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def k4_f32(self):
        return _f32([self.fx, self.fy, self.cx, self.cy])

    def k4_f64(self):
        # the fp32 values the GPU sees, widened exactly
        return _f64(self.k4_f32())


# ----------------------------------------------------------------------------------------------
# Volume (O2 allocation + O3 integration + O4 raycast)
# ----------------------------------------------------------------------------------------------
class Volume:
    """Sorted-array voxel-block volume.  See oracle.c for the algorithms."""

    def __init__(self, voxel_size=0.005, mu=0.02, w_max=100, depth_min=0.1, depth_max=10.0,
                 budget=1 << 40):
        self._L = lib()
        self.voxel_size, self.mu = float(voxel_size), float(mu)
        self.h = self._L.orc_volume_new(voxel_size, mu, int(w_max), depth_min, depth_max, int(budget))

    def __del__(self):
        try:
            self._L.orc_volume_free(self.h)
        except Exception:
            pass

    def fuse(self, cam: Camera, R, t, depth_u16: np.ndarray, depth_scale: float,
             rgba_u8: np.ndarray) -> int:
        d = np.ascontiguousarray(depth_u16, dtype=np.uint16)
        c = np.ascontiguousarray(rgba_u8, dtype=np.uint8)
        assert d.size == cam.width * cam.height and c.size == 4 * d.size
        return self._L.orc_fuse(self.h, _p(cam.k4_f32()), cam.width, cam.height,
                                _p(_f32(R).reshape(9)), _p(_f32(t).reshape(3)), _p(d),
                                float(depth_scale), _p(c))

    @property
    def n_blocks(self) -> int:
        return int(self._L.orc_volume_n(self.h))

    @property
    def overflow(self) -> bool:
        return bool(self._L.orc_volume_overflow(self.h))

    def blocks(self):
        """(coords i32[n,3] sorted lexicographically, tsdf f32[n,512], rgbw u8[n,512,4])."""
        n = self.n_blocks
        coords = np.zeros((n, 3), np.int32)
        tsdf = np.zeros((n, 512), np.float32)
        rgbw = np.zeros((n, 512, 4), np.uint8)
        self._L.orc_volume_export(self.h, _p(coords), _p(tsdf), _p(rgbw))
        return coords, tsdf, rgbw

    def visible(self):
        n = int(self._L.orc_volume_nvis(self.h))
        coords = np.zeros((n, 3), np.int32)
        self._L.orc_volume_export_visible(self.h, _p(coords))
        return coords

    def raycast(self, cam: Camera, R, t, pixels: np.ndarray | None = None):
        """O4.  pixels: int32[n,2] (u,v) or None = every pixel (row-major).
        Returns depth f64[n], color f64[n,3], vertex f64[n,3], margin f64[n]."""
        if pixels is None:
            n = cam.width * cam.height
            pp = None
        else:
            pp = np.ascontiguousarray(pixels, dtype=np.int32).reshape(-1, 2)
            n = pp.shape[0]
        depth = np.zeros(n)
        color = np.zeros((n, 3))
        vertex = np.zeros((n, 3))
        margin = np.zeros(n)
        self._L.orc_raycast(self.h, _p(cam.k4_f32()), cam.width, cam.height,
                            _p(_f32(R).reshape(9)), _p(_f32(t).reshape(3)), _p(pp), n,
                            _p(depth), _p(color), _p(vertex), _p(margin))
        return depth, color, vertex, margin


# ----------------------------------------------------------------------------------------------
# Gaussians
# ----------------------------------------------------------------------------------------------
@dataclass
class RenderCfg:
    eps_depth: float = 0.02        # R-EPS  ("a small positive threshold")
    alpha_min: float = 1.0 / 255
    near_z: float = 0.2            # R-NEAR
    lowpass: float = 0.3           # R-LOWPASS


def n_coeffs(deg: int) -> int:
    return (deg + 1) ** 2


def project_p32(g: dict, cam: Camera, R, t, cfg: RenderCfg, fields: bool = False):
    """P32 projection fields: rect i32[n,4] (x0,y0,x1,y1 inclusive), depth
    f32[n] (camera z) and culled i32[n]; with fields=True also f32[n,6] (px, py, conic a, b, c,
    ln sigma)."""
    n = int(g["xyz"].shape[0])
    rect = np.zeros((n, 4), np.int32)
    depth = np.zeros(n, np.float32)
    culled = np.zeros(n, np.int32)
    fl = np.zeros((n, 6), np.float32)
    lib().orc_project_p32_full(n, _p(_f32(g["xyz"])), _p(_f32(g["log_scale"])), _p(_f32(g["rot"])),
                               _p(_f32(g["opacity_raw"]).reshape(n)),
                               _p(cam.k4_f32()), cam.width, cam.height, _p(_f32(R).reshape(9)),
                               _p(_f32(t).reshape(3)), float(np.float32(cfg.near_z)),
                               float(np.float32(cfg.lowpass)), _p(rect), _p(depth), _p(culled), _p(fl))
    if fields:
        return rect, depth, culled, fl
    return rect, depth, culled


def tile_lists(rect, depth, culled, width: int, height: int, tile: int):
    """Plain definition of the binned, sorted lists (north_star "(tile, depth)
    key sort"): List(T) = [i : not culled, rect_i meets T] ascending by (float bits of d_i, i),
    concatenated in row-major tile order.  Returns (values u32[K], ranges u32[n_tiles, 2])."""
    tx_n = -(-width // tile)
    ty_n = -(-height // tile)
    tiles, idx = [], []
    for i in np.nonzero(culled == 0)[0]:
        x0, y0, x1, y1 = (int(v) for v in rect[i])
        for ty in range(y0 // tile, y1 // tile + 1):
            for tx in range(x0 // tile, x1 // tile + 1):
                tiles.append(ty * tx_n + tx)
                idx.append(i)
    tiles = np.asarray(tiles, np.int64)
    idx = np.asarray(idx, np.int64)
    dbits = depth.view(np.uint32)[idx].astype(np.int64) if idx.size else np.zeros(0, np.int64)
    order = np.lexsort((idx, dbits, tiles))  # primary key last
    values = idx[order].astype(np.uint32)
    counts = np.bincount(tiles, minlength=tx_n * ty_n) if tiles.size else np.zeros(tx_n * ty_n, np.int64)
    ends = np.cumsum(counts)
    ranges = np.stack([ends - counts, ends], axis=1).astype(np.uint32)
    return values, ranges


def _g64(g: dict):
    deg = int(g["sh_degree"])
    n = int(g["xyz"].shape[0])
    return (n, deg, _f64(g["xyz"]), _f64(g["log_scale"]), _f64(g["rot"]),
            _f64(g["opacity_raw"]).reshape(n), _f64(g["sh"]))


def render(g: dict, cam: Camera, R, t, Dt, Ct, cfg: RenderCfg = RenderCfg()):
    """Eqs. 1-4, F64.  Dt f[H,W] (0 = miss), Ct f[H,W,3].
    Returns dict(Cstar [H,W,3], WG [H,W], CG [H,W,3], amb bool[H,W])."""
    n, deg, xyz, ls, rot, op, sh = _g64(g)
    H, W = cam.height, cam.width
    Dt = _f64(Dt).reshape(H, W)
    Ct = _f64(Ct).reshape(H, W, 3)
    Cs = np.zeros((H, W, 3))
    WG = np.zeros((H, W))
    CG = np.zeros((H, W, 3))
    amb = np.zeros((H, W), np.uint8)
    lib().orc_render(n, deg, _p(xyz), _p(ls), _p(rot), _p(op), _p(sh), _p(cam.k4_f64()), W, H,
                     _p(_f64(_f32(R)).reshape(9)), _p(_f64(_f32(t)).reshape(3)),
                     float(np.float32(cfg.eps_depth)), float(np.float32(cfg.alpha_min)),
                     float(np.float32(cfg.near_z)), float(np.float32(cfg.lowpass)),
                     _p(Dt), _p(Ct), _p(Cs), _p(WG), _p(CG), _p(amb))
    return {"Cstar": Cs, "WG": WG, "CG": CG, "amb": amb.astype(bool)}


def l1_loss(Cstar, WG, Dt, target_rgba, amb_tol: float = 1e-5):
    """Eq. 7 with reading R-L1: mask M = {D_t > 0 or W_G > 0}; L = sum over M and the
    three channels of |C* - C_k| / (3|M|); dL/dC* = sign(C* - C_k)/(3|M|) on M (sign(0) = 0);
    empty mask -> L = 0 and zero gradient.  C_k = u8 / 255.
    Returns (loss, grad [H,W,3], mask_count, sign_ambiguous bool[H,W])."""
    Ck = np.asarray(target_rgba, np.float64)[..., :3] / 255.0
    M = (np.asarray(Dt) > 0) | (np.asarray(WG) > 0)
    cnt = int(M.sum())
    diff = np.asarray(Cstar, np.float64) - Ck
    if cnt == 0:
        return 0.0, np.zeros_like(diff), 0, np.zeros(M.shape, bool)
    loss = float(np.abs(diff)[M].sum() / (3 * cnt))
    grad = np.where(M[..., None], np.sign(diff) / (3 * cnt), 0.0)
    sign_amb = M & (np.abs(diff) < amb_tol).any(axis=-1)
    return loss, grad, cnt, sign_amb


def backward(g: dict, cam: Camera, R, t, Dt, Cstar, WG, G, cfg: RenderCfg = RenderCfg(),
             pix_amb=None):
    """Exact gradient of L w.r.t. raw parameters (reading R-GRAD), F64, given the upstream
    dL/dC* ``G`` [H,W,3] and this oracle's forward outputs.  Returns (grads dict in parameter
    SoA layout, gauss_amb bool[n])."""
    n, deg, xyz, ls, rot, op, sh = _g64(g)
    H, W = cam.height, cam.width
    out = {"xyz": np.zeros((n, 3)), "log_scale": np.zeros((n, 3)), "rot": np.zeros((n, 4)),
           "opacity_raw": np.zeros(n), "sh": np.zeros((n, n_coeffs(deg), 3))}
    gamb = np.zeros(n, np.uint8)
    pa = None if pix_amb is None else np.ascontiguousarray(pix_amb, dtype=np.uint8)
    lib().orc_backward(n, deg, _p(xyz), _p(ls), _p(rot), _p(op), _p(sh), _p(cam.k4_f64()), W, H,
                       _p(_f64(_f32(R)).reshape(9)), _p(_f64(_f32(t)).reshape(3)),
                       float(np.float32(cfg.eps_depth)), float(np.float32(cfg.alpha_min)),
                       float(np.float32(cfg.near_z)), float(np.float32(cfg.lowpass)),
                       _p(_f64(Dt).reshape(-1)), _p(_f64(Cstar).reshape(-1)), _p(_f64(WG).reshape(-1)),
                       _p(_f64(G).reshape(-1)), _p(pa), _p(out["xyz"]), _p(out["log_scale"]),
                       _p(out["rot"]), _p(out["opacity_raw"]), _p(out["sh"]), _p(gamb))
    return out, gamb.astype(bool)


# ----------------------------------------------------------------------------------------------
# Adam (O10): torch's formula, step by step, fp64.  P:157 "Libtorch"; lrs App. C P:455.
# ----------------------------------------------------------------------------------------------
@dataclass
class AdamCfg:
    lr_xyz: float = 1.6e-4
    lr_sh0: float = 2.5e-3
    lr_shrest: float = 5e-4
    lr_opacity: float = 5e-2
    lr_scale: float = 5e-3
    lr_rot: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15


def lr_groups(cfg: AdamCfg):
    return {"xyz": cfg.lr_xyz, "log_scale": cfg.lr_scale, "rot": cfg.lr_rot,
            "opacity_raw": cfg.lr_opacity, "sh0": cfg.lr_sh0, "shrest": cfg.lr_shrest}


def adam_update(p, m, v, grad, lr, step, b1, b2, eps):
    """One torch-Adam update of one tensor (fp64).  ``step`` is the new (1-based) step count.
        m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2
        p <- p - lr/(1-b1^t) * m / (sqrt(v)/sqrt(1-b2^t) + eps)"""
    m = b1 * m + (1 - b1) * grad
    v = b2 * v + (1 - b2) * grad * grad
    bc1 = 1 - b1 ** step
    bc2 = 1 - b2 ** step
    p = p - (lr / bc1) * m / (np.sqrt(v) / np.sqrt(bc2) + eps)
    return p, m, v


def adam_step(params: dict, m: dict, v: dict, grads: dict, step: int, cfg: AdamCfg = AdamCfg()):
    """Dense Adam over every parameter group (reading R-ADAM).  ``step`` = steps taken before
    this call.  SH coefficient 0 uses lr_sh0, the rest lr_shrest.  Returns new (p, m, v)."""
    t = step + 1
    lrs = lr_groups(cfg)
    P, Mo, Vo = {}, {}, {}
    for k in ("xyz", "log_scale", "rot", "opacity_raw"):
        P[k], Mo[k], Vo[k] = adam_update(_f64(params[k]), _f64(m[k]), _f64(v[k]), _f64(grads[k]),
                                         lrs[k], t, cfg.beta1, cfg.beta2, cfg.eps)
    sh = _f64(params["sh"]).copy()
    shm = _f64(m["sh"]).copy()
    shv = _f64(v["sh"]).copy()
    gsh = _f64(grads["sh"])
    n = sh.shape[0]
    sh = sh.reshape(n, -1, 3)
    shm = shm.reshape(n, -1, 3)
    shv = shv.reshape(n, -1, 3)
    gsh = gsh.reshape(n, -1, 3)
    out = [None, None, None]
    for sl, lr in ((slice(0, 1), cfg.lr_sh0), (slice(1, None), cfg.lr_shrest)):
        a, b, c = adam_update(sh[:, sl], shm[:, sl], shv[:, sl], gsh[:, sl], lr, t,
                              cfg.beta1, cfg.beta2, cfg.eps)
        sh[:, sl], shm[:, sl], shv[:, sl] = a, b, c
    P["sh"], Mo["sh"], Vo["sh"] = sh, shm, shv
    return P, Mo, Vo


def sh_basis(d):
    """Real SH basis of 3DGS (degree <= 3) at unit direction d -> (Y[16], dY[16,3])."""
    Y = np.zeros(16)
    dY = np.zeros((16, 3))
    lib().orc_sh_basis(float(d[0]), float(d[1]), float(d[2]), _p(Y), _p(dY))
    return Y, dY
