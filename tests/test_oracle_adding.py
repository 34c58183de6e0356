"""Pins of the CPU oracle for Gaussian adding and removal (oracle/adding.py; SURVEY §8(f) NEXT-2;
PAPER.md Eq. 6, App. A, Eq. 8).  Each check is fixed by
geometry, a closed form, brute force or a statistical property -- not by the oracle itself."""
import numpy as np
import pytest

from oracle import adding as A


def _plane_vertices(H=24, W=32, f=30.0, z=2.0):
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    x = (u - (W - 1) / 2) / f * z
    y = (v - (H - 1) / 2) / f * z
    return np.stack([x, y, np.full_like(x, z)], -1), np.full((H, W), z)


def test_normals_of_a_fronto_parallel_plane_face_the_camera():
    V, D = _plane_vertices()
    N = A.vertex_normals(V, D, cam_t=(0, 0, 0))
    inner = N[1:-1, 1:-1]
    assert np.allclose(inner, [0, 0, -1], atol=1e-12)
    assert np.all(N[0] == 0) and np.all(N[-1] == 0) and np.all(N[:, 0] == 0) and np.all(N[:, -1] == 0)


def test_normals_of_a_tilted_plane_and_missing_neighbours():
    rng = np.random.default_rng(0)
    n_true = np.array([0.3, -0.2, -1.0])
    n_true /= np.linalg.norm(n_true)
    V, D = _plane_vertices()
    # project the grid onto the plane n.x = n.(0,0,2) along the viewing rays (still a plane)
    d = V / np.linalg.norm(V, axis=-1, keepdims=True)
    t = (n_true @ np.array([0, 0, 2.0])) / (d @ n_true)
    V = d * t[..., None]
    D = V[..., 2].copy()
    D[5, 7] = 0.0  # a miss: it and its 4 neighbours get no normal
    N = A.vertex_normals(V, D, cam_t=(0, 0, 0))
    ok = np.abs(N).sum(-1) > 0
    assert not ok[5, 7] and not ok[5, 6] and not ok[5, 8] and not ok[4, 7] and not ok[6, 7]
    assert np.allclose(N[ok], n_true, atol=1e-9)
    assert ok.sum() == (22 * 30) - 5


def test_normal_on_a_sphere_is_radial_to_second_order():
    H = W = 41
    f, c, r = 40.0, np.array([0.0, 0.0, 1.0]), 0.3
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    d = np.stack([(u - 20) / f, (v - 20) / f, np.ones_like(u)], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    b = d @ c
    disc = b ** 2 - (c @ c - r ** 2)
    hit = disc > 0
    t = np.where(hit, b - np.sqrt(np.where(hit, disc, 0)), 0)
    V = d * t[..., None]
    N = A.vertex_normals(V, np.where(hit, V[..., 2], 0), cam_t=(0, 0, 0))
    ok = np.abs(N).sum(-1) > 0
    radial = (V - c) / r
    cosang = np.einsum("ijk,ijk->ij", N, radial)[ok]
    assert ok.sum() > 300 and cosang.min() > 0.995


def test_add_mask_thresholds_and_validity():
    H, W = 2, 3
    tgt = np.zeros((H, W, 4), np.uint8)
    tgt[..., :3] = 100
    ck = np.float32(100) * np.float32(1.0 / 255.0)
    Cs = np.full((H, W, 3), ck, np.float32)
    Cs[0, 0, 1] = ck + np.float32(0.06)  # colour error above delta_c -> in M
    Cs[0, 1, 2] = ck - np.float32(0.04)  # below -> not in M
    Cs[0, 2, 0] = ck + np.float32(0.2)   # in, but W_G = 4 -> not in M
    Cs[1, 0, 0] = ck + np.float32(0.2)   # in, but no SDF hit
    Cs[1, 1, 0] = ck + np.float32(0.2)   # in
    Cs[1, 2, 0] = ck + np.float32(0.2)   # in, but no normal
    WG = np.array([[0.0, 0.0, 4.0], [3.99, 3.99, 0.0]], np.float32)
    Dt = np.array([[1.0, 1.0, 1.0], [0.0, 1.0, 1.0]], np.float32)
    N = np.zeros((H, W, 3))
    N[..., 2] = -1
    N[1, 2] = 0
    M = A.add_mask(Cs, WG, Dt, N, tgt)
    assert M.tolist() == [[True, False, False], [False, True, False]]


def test_sampling_is_a_uniform_quarter_and_seeded():
    n = 1 << 20
    k0 = A.sample_keep(n, seed=7)
    assert abs(k0.mean() - 0.25) < 2e-3
    # uniform along the image: each of 64 stripes within 4 sigma of 25%
    stripes = k0.reshape(64, -1).mean(axis=1)
    sd = np.sqrt(0.25 * 0.75 / (n / 64))
    assert np.all(np.abs(stripes - 0.25) < 4 * sd)
    # no row-to-row correlation of the decisions
    a, b = k0[:-1].astype(float), k0[1:].astype(float)
    assert abs(np.corrcoef(a, b)[0, 1]) < 5e-3
    assert np.array_equal(k0, A.sample_keep(n, seed=7))
    assert 0.2 < (k0 != A.sample_keep(n, seed=8)).mean() < 0.5


def test_knn_scale_on_grids_and_the_cap():
    h = 0.004
    g = np.stack(np.meshgrid(np.arange(10), np.arange(10), indexing="ij"), -1).reshape(-1, 2) * h
    P = np.concatenate([g, np.zeros((100, 1))], 1)
    interior = np.flatnonzero((g[:, 0] > 0) & (g[:, 0] < 9 * h) & (g[:, 1] > 0) & (g[:, 1] < 9 * h))
    s, tie = A.knn_scale(P, interior)
    assert np.allclose(s, h, rtol=1e-12)  # 4 neighbours at h: any 3 of them give RMS h
    # a corner: neighbours at h, h, h*sqrt(2) -> RMS sqrt((1+1+2)/3) h
    s, _ = A.knn_scale(P, np.array([0]))
    assert np.isclose(s[0], h * np.sqrt(4 / 3))
    # sparse points 0.5 m apart: truncated at 0.1 (App. A)
    Q = np.arange(6)[:, None] * np.array([[0.5, 0, 0]])
    s, _ = A.knn_scale(Q, np.arange(6))
    assert np.all(s == 0.1)
    # fewer than 3 other vertices: truncated
    s, _ = A.knn_scale(Q[:3], np.arange(3))
    assert np.all(s == 0.1)


def test_knn_scale_matches_brute_force():
    rng = np.random.default_rng(3)
    P = rng.normal(size=(400, 3)) * 0.05
    q = rng.choice(400, 60, replace=False)
    s, tie = A.knn_scale(P, q)
    d = np.linalg.norm(P[q][:, None, :] - P[None, :, :], axis=-1)
    d[np.arange(60), q] = np.inf
    d3 = np.sort(d, axis=1)[:, :3]
    ref = np.minimum(np.sqrt((d3 ** 2).mean(axis=1)), 0.1)
    assert np.allclose(s, ref, rtol=1e-12)


def _rotmat(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


@pytest.mark.parametrize("n", [(0, 0, 1), (0, 0, -1), (1, 0, 0), (0.3, -0.5, -0.8), (-0.2, 0.9, 0.1)])
def test_disc_rotation_puts_the_shortest_axis_on_the_normal(n):
    n = np.array(n, np.float64) / np.linalg.norm(n)
    q = A.quat_z_to(n[None])[0]
    assert np.isclose(np.linalg.norm(q), 1.0)
    assert np.allclose(_rotmat(q) @ np.array([0, 0, 1.0]), n, atol=1e-12)


def test_init_gaussians_closed_forms():
    V, D = _plane_vertices(H=6, W=8)
    N = A.vertex_normals(V, D, (0, 0, 0))
    tgt = np.zeros((6, 8, 4), np.uint8)
    tgt[..., 0], tgt[..., 1], tgt[..., 2] = 10, 128, 250
    sel = np.zeros((6, 8), bool)
    sel[2, 3] = sel[4, 5] = True
    s1 = np.array([0.01, 0.05])
    g = A.init_gaussians(V, N, tgt, sel, s1, sh_degree=3)
    assert g["pixels"].tolist() == [2 * 8 + 3, 4 * 8 + 5]
    assert np.allclose(g["xyz"], V[[2, 4], [3, 5]])
    colour = A.C0 * g["sh"][:, :3] + 0.5  # degree-0 colour of the SH (3DGS)
    assert np.allclose(colour, np.array([10, 128, 250]) / 255.0)
    assert np.all(g["sh"][:, 3:] == 0) and g["sh"].shape == (2, 48)
    assert np.allclose(np.exp(g["log_scale"]), [[0.01, 0.01, 0.001], [0.05, 0.05, 0.005]])
    assert np.allclose(1 / (1 + np.exp(-g["opacity_raw"])), 0.5)
    for q in g["rot"]:
        assert np.allclose(_rotmat(q) @ [0, 0, 1.0], [0, 0, -1], atol=1e-12)


def test_remove_mask_examples():
    logit = lambda p: np.log(p / (1 - p))
    o = np.array([logit(0.004), logit(0.006), 0.0, 0.0, 0.0, 0.0], np.float32)
    ls = np.log(np.array([[0.01, 0.01, 0.001], [0.01, 0.01, 0.001], [0.11, 0.01, 0.001],
                          [0.05, 0.09, 0.001], [0.002, 0.0025, 0.0001], [0.0031, 0.001, 0.0001]])).astype(np.float32)
    rm = A.remove_mask(o, ls)
    assert rm.tolist() == [True, False, True, False, True, False]
    keep = ~rm
    c = A.compact({"opacity_raw": o, "log_scale": ls, "sh_degree": 3}, keep)
    assert np.array_equal(c["opacity_raw"], o[keep]) and c["sh_degree"] == 3
