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
