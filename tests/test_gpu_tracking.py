"""GPU parity of the ICP tracking (gps_track_sync; Eq. 5) against
oracle/tracking.py on the same seeded inputs: the current depth frame and the model maps V*, N*
are the generator's analytic trace (no raycast of either side).

Bars: the tracked pose within 2e-5 m and 2e-3 degrees of the oracle's (fp32 per-pixel terms and
fp32 association vs fp64: a handful of correspondences at half-pixel boundaries may differ), and
within 1 mm / 0.1 degree of the true motion; the zero-residual fixed point; the
single-plane degeneracy."""
import numpy as np
import pytest
import torch

import gps_synth as S
from oracle import tracking as OT
from tests.test_oracle_tracking import _angle_deg, _frame, _model, _rot

pytestmark = pytest.mark.gpu


def _gpu_track(G, cfg, depth_u16, V, N, Rm, tm, Ri, ti, icp=None):
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    d = torch.from_numpy(np.ascontiguousarray(depth_u16).view(np.int16)).cuda()
    Vt = torch.from_numpy(V.astype(np.float32)).cuda()
    Nt = torch.from_numpy(N.astype(np.float32)).cuda()
    return G.track(cam, d, cfg.depth_scale, Vt, Nt, Rm, tm, Ri, ti, icp)


@pytest.mark.parametrize("noise", ["none", "tof"])
def test_track_matches_oracle_and_truth(noise):
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2", noise=noise, dropout=0.0 if noise == "none" else 0.03)
    R0, t0 = S.trajectory(cfg, 1)[0]
    R0, t0 = np.asarray(R0, np.float64), np.asarray(t0, np.float64)
    R1 = _rot([0.3, 1.0, 0.2], 1.0) @ R0
    t1 = t0 + np.array([0.006, -0.005, 0.006])
    f0, f1 = _frame(cfg, R0, t0), _frame(cfg, R1, t1)
    V, N = _model(f0)
    depth = f1.depth.numpy().view(np.uint16)
    K = (cfg.fx, cfg.fy, cfg.cx, cfg.cy)
    Ro, to, info = OT.track(depth, cfg.depth_scale, K, V, N, R0, t0, R0, t0)
    res = _gpu_track(G, cfg, depth, V, N, R0, t0, R0, t0)
    assert res["converged"] and info["converged"]
    assert np.linalg.norm(res["t"] - to) < 2e-5 and _angle_deg(res["R"], Ro) < 2e-3
    tol_t, tol_a = (1e-3, 0.1) if noise == "none" else (3e-3, 0.2)
    assert np.linalg.norm(res["t"] - t1) < tol_t and _angle_deg(res["R"], R1) < tol_a
    assert abs(res["inlier_frac"] - info["inlier_frac"]) < 1e-3


def test_track_zero_residual_fixed_point():
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2", noise="none", dropout=0.0)
    R0, t0 = S.trajectory(cfg, 1)[0]
    f0 = _frame(cfg, R0, t0)
    V, N = _model(f0)
    res = _gpu_track(G, cfg, f0.depth.numpy().view(np.uint16), V, N, R0, t0, R0, t0)
    assert res["converged"] and res["inlier_frac"] > 0.9
    assert np.linalg.norm(res["t"] - np.asarray(t0, np.float64)) < 1e-5
    assert _angle_deg(res["R"], np.asarray(R0, np.float64)) < 1e-3


def test_track_single_plane_is_degenerate():
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg1")
    H, W = cfg.height, cfg.width
    d = np.full((H, W), 2.0)
    V = OT.backproject(d, cfg.fx, cfg.fy, cfg.cx, cfg.cy)
    N = np.zeros_like(V)
    N[..., 2] = -1
    depth = np.round(d * cfg.depth_scale).astype(np.uint16)
    icp = G.IcpConfig(levels=1, iters=(3,))
    res = _gpu_track(G, cfg, depth, V, N, np.eye(3), np.zeros(3), np.eye(3), np.zeros(3), icp)
    assert res["degenerate"] and not res["converged"]
    assert np.allclose(res["R"], np.eye(3)) and np.allclose(res["t"], 0)
