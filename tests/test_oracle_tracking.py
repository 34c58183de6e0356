"""Pins of the CPU ICP oracle (oracle/tracking.py; Eq. 5; SPEC S:205-254 examples):
zero-residual fixed point, recovery of a known synthetic motion, left-invariance under a global
rigid transform, the rank deficiency of a single plane, the SE(3) exponential.  Model maps are the
generator's analytic hit points and normals -- no raycast of either implementation."""
import numpy as np
import pytest

import gps_synth as S
from oracle import tracking as T


def _rot(axis, deg):
    a = np.asarray(axis, np.float64)
    a /= np.linalg.norm(a)
    R, _ = T.exp_se3(np.concatenate([np.zeros(3), a * np.radians(deg)]))
    return R


def _frame(cfg, R, t):
    scene = S.make_scene(cfg)
    return S.render_frame(cfg, scene, np.asarray(R, np.float32), np.asarray(t, np.float32))


def _model(fr):
    """Model maps V*, N* (world) from the analytic trace, normals turned to the camera."""
    V = fr.points.numpy().astype(np.float64)
    N = fr.normal.numpy().astype(np.float64)
    hit = fr.depth_m.numpy() > 0
    flip = np.einsum("ijk,ijk->ij", N, V - fr.t.astype(np.float64)) > 0
    N = np.where(flip[..., None], -N, N)
    V[~hit] = 0
    N[~hit] = 0
    return V, N


@pytest.fixture(scope="module")
def seq():
    cfg = S.get_config("cfg2", noise="none", dropout=0.0)
    R0, t0 = S.trajectory(cfg, 1)[0]
    R0, t0 = np.asarray(R0, np.float64), np.asarray(t0, np.float64)
    # true motion of the next frame: 1 degree about a tilted axis + 1 cm
    R1 = _rot([0.3, 1.0, 0.2], 1.0) @ R0
    t1 = t0 + np.array([0.006, -0.005, 0.006])
    f0, f1 = _frame(cfg, R0, t0), _frame(cfg, R1, t1)
    K = (cfg.fx, cfg.fy, cfg.cx, cfg.cy)
    return cfg, K, (R0, t0, f0), (R1, t1, f1)


def _angle_deg(Ra, Rb):
    # ||Ra - Rb||_F = 2 sqrt(2) sin(theta / 2): accurate near 0, unlike arccos of the trace
    return np.degrees(2 * np.arcsin(min(1.0, np.linalg.norm(Ra - Rb) / (2 * np.sqrt(2)))))


def test_zero_residual_fixed_point(seq):
    cfg, K, (R0, t0, f0), _ = seq
    V, N = _model(f0)
    R, t, info = T.track(f0.depth.numpy().view(np.uint16), cfg.depth_scale, K, V, N, R0, t0, R0, t0)
    assert info["converged"] and info["inlier_frac"] > 0.9
    assert np.linalg.norm(t - t0) < 1e-6 and _angle_deg(R, R0) < np.degrees(1e-5)


def test_recovers_a_known_motion(seq):
    cfg, K, (R0, t0, f0), (R1, t1, f1) = seq
    V, N = _model(f0)
    R, t, info = T.track(f1.depth.numpy().view(np.uint16), cfg.depth_scale, K, V, N, R0, t0, R0, t0)
    assert info["converged"]
    assert np.linalg.norm(t - t1) < 1e-3 and _angle_deg(R, R1) < 0.1
    # and much closer than the start
    assert np.linalg.norm(t - t1) < 0.1 * np.linalg.norm(t0 - t1)


def test_left_invariance(seq):
    cfg, K, (R0, t0, f0), (R1, t1, f1) = seq
    V, N = _model(f0)
    depth = f1.depth.numpy().view(np.uint16)
    Ra, ta, _ = T.track(depth, cfg.depth_scale, K, V, N, R0, t0, R0, t0)
    Gr, Gt = _rot([1, -2, 0.5], 37.0), np.array([1.5, -0.7, 2.0])
    Vg = np.where(np.abs(V).sum(-1, keepdims=True) > 0, V @ Gr.T + Gt, 0)
    Ng = N @ Gr.T
    Rb, tb, _ = T.track(depth, cfg.depth_scale, K, Vg, Ng, Gr @ R0, Gr @ t0 + Gt, Gr @ R0, Gr @ t0 + Gt)
    assert np.allclose(Rb, Gr @ Ra, atol=1e-6) and np.allclose(tb, Gr @ ta + Gt, atol=1e-6)


def test_single_plane_is_degenerate():
    H, W, f = 48, 64, 60.0
    K = (f, f, 31.5, 23.5)
    d = np.full((H, W), 2.0)
    depth = np.round(d * 1000).astype(np.uint16)
    V = T.backproject(d, *K)
    N = np.zeros_like(V)
    N[..., 2] = -1
    R, t, info = T.track(depth, 1000.0, K, V, N, np.eye(3), np.zeros(3), np.eye(3), np.zeros(3), T.IcpCfg(levels=1, iters=(3,)))
    assert info["degenerate"] and not info["converged"]
    assert np.allclose(R, np.eye(3)) and np.allclose(t, 0)


def test_exp_se3_is_a_rotation_and_first_order_exact():
    xi = np.array([0.01, -0.02, 0.03, 0.2, -0.1, 0.05])
    R, v = T.exp_se3(xi)
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12) and np.isclose(np.linalg.det(R), 1)
    assert np.allclose(v, xi[:3])
    small = xi * 1e-6
    Rs, _ = T.exp_se3(small)
    p = np.array([0.3, -1.0, 2.0])
    assert np.allclose(Rs @ p, p + np.cross(small[3:], p), atol=1e-15)


def test_pyramid_averages_valid_children_only():
    d = np.array([[1.0, 0.0, 2.0, 2.0], [3.0, 0.0, 2.0, 20.0]])
    pyr = T.depth_pyramid(d, 2, 0.1, 10.0)
    assert np.allclose(pyr[1], [[2.0, 2.0]])  # (1+3)/2 ; 20 m is out of range
    fx, fy, cx, cy = T.level_intrinsics(600, 600, 319.5, 239.5, 1)
    assert (fx, cx, cy) == (300, 159.5, 119.5)


def _bilateral_brute(d, r, ss, sr):
    """The R-ICP-FILT definition with plain loops (tiny inputs only)."""
    H, W = d.shape
    out = np.zeros_like(d)
    for y in range(H):
        for x in range(W):
            if d[y, x] <= 0:
                continue
            sw = sz = 0.0
            for yy in range(max(0, y - r), min(H, y + r + 1)):
                for xx in range(max(0, x - r), min(W, x + r + 1)):
                    if d[yy, xx] > 0:
                        w = np.exp(-((xx - x) ** 2 + (yy - y) ** 2) / (2 * ss * ss)
                                   - (d[yy, xx] - d[y, x]) ** 2 / (2 * sr * sr))
                        sw += w
                        sz += w * d[yy, xx]
            out[y, x] = sz / sw
    return out


def test_bilateral_matches_its_definition_and_special_cases():
    rng = np.random.default_rng(3)
    d = 2.0 + 0.02 * rng.standard_normal((9, 11))
    d[rng.random(d.shape) < 0.2] = 0.0  # invalid pixels
    assert np.allclose(T.bilateral(d, 2, 1.5, 0.03), _bilateral_brute(d, 2, 1.5, 0.03), rtol=0, atol=1e-14)
    # constant depth is a fixed point; invalid pixels stay invalid, valid ones stay valid
    c = np.full((6, 7), 1.7)
    c[2, 3] = 0.0
    f = T.bilateral(c, 3, 4.5, 0.03)
    assert f[2, 3] == 0.0 and np.allclose(np.delete(f.ravel(), 2 * 7 + 3), 1.7, rtol=0, atol=1e-15)
    # a 1 m step is preserved (range weight exp(-1 / (2 * 0.03^2)) underflows)
    s = np.ones((5, 8))
    s[:, 4:] = 2.0
    assert np.array_equal(T.bilateral(s, 3, 4.5, 0.03), s)
    # noise is reduced on a plane
    n = 2.0 + 0.01 * rng.standard_normal((40, 40))
    assert np.std(T.bilateral(n, 3, 4.5, 0.03)[5:-5, 5:-5] - 2.0) < 0.5 * np.std(n - 2.0)


def test_filtered_track_recovers_a_known_motion():
    """R-ICP-FILT on ToF-noisy depth (cfg2): the filtered ICP recovers the true motion, closer
    than the unfiltered one, with most valid pixels kept as inliers."""
    cfg = S.get_config("cfg2", noise="tof", dropout=0.0)
    R0, t0 = S.trajectory(cfg, 1)[0]
    R0, t0 = np.asarray(R0, np.float64), np.asarray(t0, np.float64)
    R1 = _rot([0.3, 1.0, 0.2], 0.5) @ R0
    t1 = t0 + np.array([0.004, -0.003, 0.002])
    f0 = _frame(S.get_config("cfg2", noise="none", dropout=0.0), R0, t0)
    f1 = _frame(cfg, R1, t1)
    V, N = _model(f0)
    K = (cfg.fx, cfg.fy, cfg.cx, cfg.cy)
    d = f1.depth.numpy().view(np.uint16)
    R, t, info = T.track(d, cfg.depth_scale, K, V, N, R0, t0, R0, t0, T.IcpCfg(filter_radius=3))
    Ru, tu, _ = T.track(d, cfg.depth_scale, K, V, N, R0, t0, R0, t0, T.IcpCfg(filter_radius=0))
    assert info["converged"] and info["inlier_frac"] > 0.9 and info["pivot_ratio"] > 1e-3
    assert np.linalg.norm(t - t1) < 2e-4 and _angle_deg(R, R1) < 0.01
    assert np.linalg.norm(t - t1) < np.linalg.norm(tu - t1)
