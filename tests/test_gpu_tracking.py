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
    # R-ICP-FAIL: the failed frame keeps its initial pose (bit for bit)
    Ri, ti = _rot([0.0, 0.0, 1.0], 2.0).astype(np.float32), np.array([0.01, 0.0, 0.0], np.float32)
    res = _gpu_track(G, cfg, depth, V, N, np.eye(3), np.zeros(3), Ri, ti, icp)
    assert res["degenerate"] and np.array_equal(res["T"][0], Ri) and np.array_equal(res["T"][1], ti)
    res = _gpu_track(G, cfg, depth, V, N, np.eye(3), np.zeros(3), Ri, ti, G.IcpConfig(levels=1, iters=(3,),
                                                                                  fallback=False))
    assert np.array_equal(res["T"][0], res["R"].astype(np.float32))


def test_pose_extrapolate_is_constant_velocity():
    """gps_pose_extrapolate: T_b (T_a^-1 T_b) against the same product in fp64 numpy."""
    import paper_2509_11574_b200 as G
    rng = np.random.default_rng(5)
    for _ in range(5):
        Ra = _rot(rng.normal(size=3), rng.uniform(0, 180))
        Rb = _rot(rng.normal(size=3), rng.uniform(0, 180))
        ta, tb = rng.normal(size=3), rng.normal(size=3)
        Ta, Tb = np.eye(4), np.eye(4)
        Ta[:3, :3], Ta[:3, 3] = Ra, ta
        Tb[:3, :3], Tb[:3, 3] = Rb, tb
        ref = Tb @ np.linalg.inv(Ta) @ Tb
        a = G.pose_tensor(Ra.astype(np.float32), ta.astype(np.float32))
        b = G.pose_tensor(Rb.astype(np.float32), tb.astype(np.float32))
        out = torch.empty(12, dtype=torch.float32, device="cuda")
        o = G.pose_extrapolate(a, b, out).cpu().numpy().astype(np.float64)
        assert np.abs(o[:9] - ref[:3, :3].reshape(9)).max() < 2e-6
        assert np.abs(o[9:] - ref[:3, 3]).max() < 2e-5


def test_track_async_equals_sync_bitwise():
    """gps_track_async (device poses, no synchronisation) runs the kernels of gps_track_sync: the
    same pose bits and the same result record; the initial pose may alias the output."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2", noise="tof", dropout=0.03)
    R0, t0 = S.trajectory(cfg, 1)[0]
    R0, t0 = np.asarray(R0, np.float64), np.asarray(t0, np.float64)
    R1 = _rot([0.3, 1.0, 0.2], 1.0) @ R0
    t1 = t0 + np.array([0.006, -0.005, 0.006])
    f0, f1 = _frame(cfg, R0, t0), _frame(cfg, R1, t1)
    V, N = _model(f0)
    depth = f1.depth.numpy().view(np.uint16)
    ref = _gpu_track(G, cfg, depth, V, N, R0, t0, R0, t0)
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    d = torch.from_numpy(np.ascontiguousarray(depth).view(np.int16)).cuda()
    Vt = torch.from_numpy(V.astype(np.float32)).cuda()
    Nt = torch.from_numpy(N.astype(np.float32)).cuda()
    pose = G.pose_tensor(R0, t0)
    raw = torch.zeros(G.TRACK_RESULT_BYTES, dtype=torch.uint8, device="cuda")
    G.track_async(cam, d, cfg.depth_scale, Vt, Nt, pose, pose, pose, raw)  # in place
    res = G.track_result(raw)
    assert np.array_equal(res["R"], ref["R"]) and np.array_equal(res["t"], ref["t"])
    assert res["steps"] == ref["steps"] and res["inliers"] == ref["inliers"] and res["energy"] == ref["energy"]
    host = pose.cpu().numpy()
    assert np.array_equal(host[:9], ref["R"].astype(np.float32).reshape(9))
    assert np.array_equal(host[9:], ref["t"].astype(np.float32))


def test_dpose_forms_equal_host_pose_forms_bitwise():
    """gps_fuse_dpose / gps_raycast_dpose / gps_vertex_normals_dpose read the pose on the device
    and otherwise run the kernels of the host-pose forms: bit-identical volumes and maps."""
    import paper_2509_11574_b200 as G
    from tests import gpu_helpers as H
    cfg = S.get_config("cfg2")
    frs = H.frames(cfg, 3)
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    vols = [H.gpu_volume(cfg) for _ in range(2)]
    for fr in frs:
        d, c = fr.depth.cuda(), fr.rgba.cuda()
        vols[0].fuse(cam, fr.R, fr.t, d, cfg.depth_scale, c)
        vols[1].fuse_dpose(cam, G.pose_tensor(fr.R, fr.t), d, cfg.depth_scale, c)
    ca, va = vols[0].export_blocks()
    cb, vb = vols[1].export_blocks()
    ca, va = H.sorted_blocks(ca, va)
    cb, vb = H.sorted_blocks(cb, vb)
    assert len(ca) > 100 and np.array_equal(ca, cb) and np.array_equal(va.view(np.uint8), vb.view(np.uint8))
    fr = frs[-1]
    H_, W_ = cfg.height, cfg.width
    outs = []
    for k, vol in enumerate(vols):
        dep = torch.empty((H_, W_), dtype=torch.float32, device="cuda")
        col = torch.empty((H_, W_, 3), dtype=torch.float32, device="cuda")
        ver = torch.empty((H_, W_, 3), dtype=torch.float32, device="cuda")
        nor = torch.empty((H_, W_, 3), dtype=torch.float32, device="cuda")
        if k == 0:
            vol.raycast(cam, fr.R, fr.t, dep, col, ver)
            G.vertex_normals(cam, fr.R, fr.t, dep, ver, out=nor)
        else:
            p = G.pose_tensor(fr.R, fr.t)
            vol.raycast_dpose(cam, p, dep, col, ver)
            G.vertex_normals_dpose(cam, p, dep, ver, nor)
        outs.append([x.cpu().numpy() for x in (dep, col, ver, nor)])
    assert (outs[0][0] > 0).mean() > 0.5
    for a, b in zip(*outs):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_track_from_a_predicted_init_matches_oracle():
    """T_init != T_model (the constant-velocity prediction of the pipeline): association still
    uses T_model's camera (Eq. 5); the GPU and the oracle reach the same pose, and the same as
    from T_init = T_model."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2", noise="none", dropout=0.0)
    R0, t0 = S.trajectory(cfg, 1)[0]
    R0, t0 = np.asarray(R0, np.float64), np.asarray(t0, np.float64)
    R1 = _rot([0.3, 1.0, 0.2], 0.3) @ R0
    t1 = t0 + np.array([0.006, -0.005, 0.003])
    Ri, ti = _rot([0.3, 1.0, 0.2], 0.3) @ R1, t1 + (t1 - t0)
    f0, f1 = _frame(cfg, R0, t0), _frame(cfg, R1, t1)
    V, N = _model(f0)
    depth = f1.depth.numpy().view(np.uint16)
    K = (cfg.fx, cfg.fy, cfg.cx, cfg.cy)
    Ro, to, info = OT.track(depth, cfg.depth_scale, K, V, N, R0, t0, Ri, ti)
    res = _gpu_track(G, cfg, depth, V, N, R0, t0, Ri, ti)
    ref = _gpu_track(G, cfg, depth, V, N, R0, t0, R0, t0)
    assert res["converged"] and info["converged"]
    assert np.linalg.norm(res["t"] - to) < 2e-5 and _angle_deg(res["R"], Ro) < 2e-3
    assert np.linalg.norm(res["t"] - ref["t"]) < 2e-5 and _angle_deg(res["R"], ref["R"]) < 2e-3


def test_chained_pose_predictions_stay_rigid():
    """Chained constant-velocity predictions (every frame's ICP failing) follow the exact screw
    motion and stay orthonormal: no growth of the fp32 rounding (the extrapolation re-orthonormalises)."""
    import paper_2509_11574_b200 as G
    w = _rot([0.2, 1.0, -0.3], 0.7)
    v = np.array([0.004, -0.002, 0.007])
    poses = [G.pose_tensor(np.eye(3, dtype=np.float32), np.zeros(3, np.float32)),
             G.pose_tensor(w.astype(np.float32), v.astype(np.float32))]
    for _ in range(60):
        poses.append(G.pose_extrapolate(poses[-2], poses[-1], torch.empty(12, dtype=torch.float32, device="cuda")))
    o = poses[-1].cpu().numpy().astype(np.float64)
    D = np.eye(4)
    D[:3, :3], D[:3, 3] = w, v
    ref = np.linalg.matrix_power(D, 61)
    R = o[:9].reshape(3, 3)
    assert np.abs(R @ R.T - np.eye(3)).max() < 1e-6
    assert np.abs(R - ref[:3, :3]).max() < 1e-4 and np.abs(o[9:] - ref[:3, 3]).max() < 1e-4


def test_filtered_track_matches_oracle():
    """R-ICP-FILT (bilateral pre-filter of the tracking depth, k_icp_bilateral) on ToF-noisy cfg2:
    GPU pose = oracle pose within the tracking bars; the same convergence decision."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2", noise="tof", dropout=0.03)
    R0, t0 = S.trajectory(cfg, 1)[0]
    R0, t0 = np.asarray(R0, np.float64), np.asarray(t0, np.float64)
    R1 = _rot([0.3, 1.0, 0.2], 0.5) @ R0
    t1 = t0 + np.array([0.004, -0.003, 0.002])
    f0, f1 = _frame(S.get_config("cfg2", noise="none", dropout=0.0), R0, t0), _frame(cfg, R1, t1)
    V, N = _model(f0)
    depth = f1.depth.numpy().view(np.uint16)
    K = (cfg.fx, cfg.fy, cfg.cx, cfg.cy)
    Ro, to, info = OT.track(depth, cfg.depth_scale, K, V, N, R0, t0, R0, t0, OT.IcpCfg(filter_radius=3))
    res = _gpu_track(G, cfg, depth, V, N, R0, t0, R0, t0, G.IcpConfig(filter_radius=3))
    assert res["converged"] and info["converged"]
    assert np.linalg.norm(res["t"] - to) < 2e-5 and _angle_deg(res["R"], Ro) < 2e-3
    assert abs(res["inlier_frac"] - info["inlier_frac"]) < 2e-3
    assert abs(res["pivot_ratio"] - info["pivot_ratio"]) < 1e-3 * info["pivot_ratio"] + 1e-6


def test_track_full_size_cfg4():
    """The pipeline's tracking configuration (R-ICP-FILT on) at the bench's full 1280x720 on the
    ToF-noisy cfg4 sensor model: GPU pose = oracle pose within the tracking bars."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg4")
    R0, t0 = S.trajectory(cfg, 1)[0]
    R0, t0 = np.asarray(R0, np.float64), np.asarray(t0, np.float64)
    R1 = _rot([0.2, 1.0, -0.1], 0.4) @ R0
    t1 = t0 + np.array([0.005, 0.002, -0.004])
    f0, f1 = _frame(S.get_config("cfg4", noise="none", dropout=0.0), R0, t0), _frame(cfg, R1, t1)
    V, N = _model(f0)
    depth = f1.depth.numpy().view(np.uint16)
    K = (cfg.fx, cfg.fy, cfg.cx, cfg.cy)
    Ro, to, info = OT.track(depth, cfg.depth_scale, K, V, N, R0, t0, R0, t0, OT.IcpCfg(filter_radius=3))
    res = _gpu_track(G, cfg, depth, V, N, R0, t0, R0, t0, G.IcpConfig(filter_radius=3))
    assert res["converged"] == info["converged"] and res["converged"]
    assert np.linalg.norm(res["t"] - to) < 2e-5 and _angle_deg(res["R"], Ro) < 2e-3
    assert np.linalg.norm(res["t"] - t1) < 2e-3 and _angle_deg(res["R"], R1) < 0.1
