"""Pins of the oracle's Gaussian path: projection ("following 3DGS"), Eqs. 1-4
(P:75-97), the L1 loss (Eq. 7) and its exact gradient, against closed forms,
worked examples, invariants, an independent all-pairs torch implementation
differentiated by autograd, and fp64 finite differences.  Readings R-FOOT, R-EPS, R-MISS,
R-SH, R-QUAT, R-NEAR, R-LOWPASS, R-L1, R-GRAD in DESIGN.md §3."""
import numpy as np
import pytest
import torch

import oracle as O
from gps_synth import random_gaussians
from tests import refimpl as RI

CFG = O.RenderCfg()


def small_cam(w=32, h=24, f=30.0, cx=None, cy=None):
    return O.Camera(f, f, (w - 1) / 2 if cx is None else cx, (h - 1) / 2 if cy is None else cy, w, h)


def one_gaussian(p, s, q=(1, 0, 0, 0), o=0.0, sh0=(0.0, 0.0, 0.0), deg=0):
    nc = (deg + 1) ** 2
    sh = np.zeros((1, nc * 3), np.float32)
    sh[0, :3] = sh0
    return {"sh_degree": deg, "xyz": np.array([p], np.float32),
            "log_scale": np.log(np.array([s], np.float32)).astype(np.float32),
            "rot": np.array([q], np.float32), "opacity_raw": np.array([o], np.float32), "sh": sh}


def cam_tuple(c):
    return (c.fx, c.fy, c.cx, c.cy, c.width, c.height)


# ---------------------------------------------------------------------------------------------
def test_sh_basis_orthonormal_and_derivatives():
    """The degree<=3 real SH basis is orthonormal on the sphere: Gauss-Legendre x uniform-phi
    quadrature (exact for these polynomials) gives the identity to 1e-12.  This pins every SH
    constant (R-SH).  dY matches central differences."""
    xg, wg = np.polynomial.legendre.leggauss(24)
    phis = np.linspace(0, 2 * np.pi, 48, endpoint=False)
    G = np.zeros((16, 16))
    for ct, w in zip(xg, wg):
        st = np.sqrt(1 - ct * ct)
        for ph in phis:
            Y, _ = O.sh_basis((st * np.cos(ph), st * np.sin(ph), ct))
            G += w * (2 * np.pi / len(phis)) * np.outer(Y, Y)
    assert np.max(np.abs(G - np.eye(16))) < 1e-12
    d = np.array([0.3, -0.5, 0.81])
    _, dY = O.sh_basis(d)
    for e in range(3):
        h = np.zeros(3)
        h[e] = 1e-6
        fd = (O.sh_basis(d + h)[0] - O.sh_basis(d - h)[0]) / 2e-6
        assert np.max(np.abs(fd - dY[:, e])) < 1e-8


@pytest.mark.parametrize("fx", [40.0, 80.0])
def test_on_axis_isotropic_closed_form(fx):
    """an isotropic Gaussian on the optical axis projects to p_hat = (cx, cy) with
    Sigma_2D = ((fx s/z)^2 + 0.3) I, for any rotation q; so W_G at pixel (cx+k, cy) equals
    sigma exp(-k^2 / (2 v)) exactly where the pair is in (Eq. 3, R-LOWPASS, R-FOOT)."""
    c = small_cam(41, 31, fx, cx=20.0, cy=15.0)
    z, s = 1.0, 0.02
    for q in ((1, 0, 0, 0), (0.3, -0.5, 0.7, 0.2)):
        g = one_gaussian((0, 0, z), (s, s, s), q, o=1.0)
        Dt = np.zeros((c.height, c.width))
        Ct = np.zeros((c.height, c.width, 3))
        out = O.render(g, c, np.eye(3), np.zeros(3), Dt, Ct)
        se = np.exp(np.float64(g["log_scale"][0, 0]))  # the stored (fp32) scale
        v = (fx * se / z) ** 2 + np.float64(np.float32(0.3))
        sig = 1 / (1 + np.exp(-1.0))
        for k in range(0, 8):
            qf = k * k / v
            a = sig * np.exp(-0.5 * qf)
            expect = a if (qf <= 9 and a >= 1 / 255) else 0.0
            assert abs(out["WG"][15, 20 + k] - expect) < 1e-12
            assert abs(out["WG"][15 + k, 20] - expect) < 1e-12


def test_zero_gaussians_identity():
    """AC1: with no Gaussians C* = C_t exactly."""
    c = small_cam()
    rng = np.random.default_rng(0)
    g = random_gaussians(0, 1, rng)
    Ct = rng.random((c.height, c.width, 3))
    Dt = rng.uniform(0, 2, (c.height, c.width))
    out = O.render(g, c, np.eye(3), np.zeros(3), Dt, Ct)
    assert np.array_equal(out["Cstar"], Ct) and np.all(out["WG"] == 0)


def test_single_gaussian_centre_pixel():
    """one Gaussian centred on an integer pixel with sigma = 0.5: alpha = 0.5,
    W_G = 0.5, C_G = 0.5 c, C* = (C_t + 0.5 c)/1.5.  sh0 = 0 gives c = 0.5 exactly."""
    c = small_cam(33, 25, 30.0, cx=16.0, cy=12.0)
    g = one_gaussian((0, 0, 1.0), (0.01, 0.01, 0.01), o=0.0)
    Ct = np.full((c.height, c.width, 3), 0.2)
    out = O.render(g, c, np.eye(3), np.zeros(3), np.zeros((c.height, c.width)), Ct)
    assert out["WG"][12, 16] == 0.5
    assert np.allclose(out["CG"][12, 16], 0.25, atol=0, rtol=0)
    assert np.allclose(out["Cstar"][12, 16], (0.2 + 0.25) / 1.5, atol=1e-15)


def test_behind_wall_contributes_exactly_zero():
    """AC4: a Gaussian 10 cm behind the SDF surface (eps = 2 cm) adds exactly 0
    everywhere and receives exactly zero gradient (Eq. 1 indicator, R-GRAD)."""
    c = small_cam()
    g = one_gaussian((0.01, 0.0, 1.1), (0.03, 0.03, 0.03), o=2.0, sh0=(1.0, 0.5, -0.3))
    Dt = np.full((c.height, c.width), 1.0)
    Ct = np.full((c.height, c.width, 3), 0.3)
    out = O.render(g, c, np.eye(3), np.zeros(3), Dt, Ct)
    assert np.all(out["WG"] == 0) and np.array_equal(out["Cstar"], Ct)
    G = np.random.default_rng(1).normal(size=(c.height, c.width, 3))
    grads, _ = O.backward(g, c, np.eye(3), np.zeros(3), Dt, out["Cstar"], out["WG"], G)
    for v in grads.values():
        assert np.all(v == 0)
    # the same Gaussian in front of the wall does contribute
    g2 = one_gaussian((0.01, 0.0, 0.9), (0.03, 0.03, 0.03), o=2.0)
    assert O.render(g2, c, np.eye(3), np.zeros(3), Dt, Ct)["WG"].max() > 0.5


def scene(seed, n=6, deg=3, w=32, h=24):
    rng = np.random.default_rng(seed)
    c = small_cam(w, h, 30.0)
    R = RI.random_rotation(rng) if seed % 2 else np.eye(3, dtype=np.float32)
    t = rng.uniform(-0.05, 0.05, 3).astype(np.float32)
    ctr = R.astype(np.float64) @ np.array([0, 0, 1.0]) + t
    g = random_gaussians(n, deg, rng, center=ctr, spread=0.12, scale=(0.01, 0.06))
    Dt = rng.uniform(0.9, 1.15, (h, w))
    Dt[rng.random((h, w)) < 0.1] = 0.0
    Ct = rng.random((h, w, 3))
    return c, R, t, g, Dt, Ct, rng


@pytest.mark.parametrize("seed", range(6))
def test_forward_matches_independent_allpairs(seed):
    """Brute force: the oracle (per-Gaussian rect loops, C) equals an independent all-pairs
    torch implementation (matrix algebra, quaternion sandwich) to 1e-10 on unambiguous pixels."""
    c, R, t, g, Dt, Ct, _ = scene(seed)
    out = O.render(g, c, R, t, Dt, Ct)
    Cs, WG, _ = RI.render_allpairs(RI.to_torch_params(g), cam_tuple(c), R, t, Dt, Ct)
    ok = ~out["amb"]
    assert ok.mean() > 0.99
    assert np.max(np.abs(out["Cstar"][ok] - Cs.numpy()[ok])) < 1e-10
    assert np.max(np.abs(out["WG"][ok] - WG.numpy()[ok])) < 1e-10
    assert out["WG"].max() > 0.1  # the scene is not empty


def test_permutation_invariance_and_epsilon_monotonicity():
    """AC2: C* is order independent (<= 1e-12 in fp64).  S:340: decreasing eps never
    increases W_G.  S:343: C* is a convex combination of C_t and C_G/W_G."""
    c, R, t, g, Dt, Ct, rng = scene(7, n=40)
    out = O.render(g, c, R, t, Dt, Ct)
    perm = rng.permutation(40)
    gp = {k: (v[perm] if isinstance(v, np.ndarray) else v) for k, v in g.items()}
    outp = O.render(gp, c, R, t, Dt, Ct)
    assert np.max(np.abs(out["Cstar"] - outp["Cstar"])) < 1e-12
    small = O.render(g, c, R, t, Dt, Ct, O.RenderCfg(eps_depth=0.005))
    assert np.all(small["WG"] <= out["WG"] + 1e-15)
    W = out["WG"]
    has = W > 0
    gm = out["CG"][has] / W[has][:, None]
    lo = np.minimum(Ct[has], gm) - 1e-12
    hi = np.maximum(Ct[has], gm) + 1e-12
    assert np.all((out["Cstar"][has] >= lo) & (out["Cstar"][has] <= hi))


def test_l1_worked_example():
    """a single pixel with C* - C_k = (0.1, -0.1, 0) gives L = 0.2/3 and gradient signs
    (+, -, 0); C* = C_k gives 0; an empty mask gives 0 and zero gradient."""
    tgt = np.array([[[100, 100, 100, 255]]], np.uint8)
    Ck = 100 / 255.0
    Cs = np.array([[[Ck + 0.1, Ck - 0.1, Ck]]])
    loss, grad, cnt, _ = O.l1_loss(Cs, np.zeros((1, 1)), np.ones((1, 1)), tgt)
    assert cnt == 1 and abs(loss - 0.2 / 3) < 1e-15
    assert np.array_equal(np.sign(grad[0, 0]), [1, -1, 0])
    assert O.l1_loss(np.full((1, 1, 3), Ck), np.zeros((1, 1)), np.ones((1, 1)), tgt)[0] == 0
    l0, g0, c0, _ = O.l1_loss(Cs, np.zeros((1, 1)), np.zeros((1, 1)), tgt)
    assert l0 == 0 and c0 == 0 and np.all(g0 == 0)


def test_l1_mask_includes_gaussian_only_pixels():
    """R-L1 mask M = {D_t > 0 or W_G > 0} (P:15 Gaussians fill "missing data"): a pixel
    the SDF missed (D_t = 0) but a Gaussian covers (W_G > 0) is in the loss and gets a
    gradient; a pixel with neither is not.  Three pixels, hand-computed:
    |C* - C_k| sums 0.3 (SDF hit) + 1.2 (Gaussian only) over |M| = 2 -> L = 1.5/6 = 0.25."""
    tgt = np.zeros((1, 3, 4), np.uint8)
    Cs = np.array([[[0.1] * 3, [0.4] * 3, [0.9] * 3]])
    Dt = np.array([[0.5, 0.0, 0.0]])
    WG = np.array([[0.0, 0.3, 0.0]])
    loss, grad, cnt, _ = O.l1_loss(Cs, WG, Dt, tgt)
    assert cnt == 2
    assert abs(loss - 0.25) < 1e-15
    assert np.allclose(grad[0, 0], 1 / 6) and np.allclose(grad[0, 1], 1 / 6)
    assert np.all(grad[0, 2] == 0)


GROUPS = ("xyz", "log_scale", "rot", "opacity_raw", "sh")


@pytest.mark.parametrize("seed", range(8))
def test_backward_equals_autograd_of_independent_forward(seed):
    """R-GRAD: the oracle's hand-derived chain rule equals torch.autograd (fp64) through the
    independent all-pairs forward, for a random linear upstream dL/dC* (1e-9 relative)."""
    c, R, t, g, Dt, Ct, rng = scene(100 + seed, n=int(rng_n(seed)))
    G = rng.normal(size=(c.height, c.width, 3))
    out = O.render(g, c, R, t, Dt, Ct)
    grads, gamb = O.backward(g, c, R, t, Dt, out["Cstar"], out["WG"], G, pix_amb=out["amb"])
    tp = RI.to_torch_params(g, requires_grad=True)
    Cs, _, _ = RI.render_allpairs(tp, cam_tuple(c), R, t, Dt, Ct)
    (Cs * torch.as_tensor(G)).sum().backward()
    keep = ~gamb
    for k in GROUPS:
        ref = tp[k].grad.numpy().reshape(grads[k].shape)
        a, b = grads[k][keep], ref[keep]
        scale = max(np.max(np.abs(b)), 1e-300)
        assert np.max(np.abs(a - b)) <= 1e-9 * scale, k


def rng_n(seed):
    return [1, 2, 3, 5, 8, 8, 4, 6][seed]


@pytest.mark.parametrize("seed", range(5))
def test_backward_matches_finite_differences(seed):
    """AC3: central differences in fp64 of L_r = sum r C* (linear upstream avoids the
    L1 kink) on every raw parameter; parameters whose in-pair set changes between theta +- h
    are skipped (membership change detection)."""
    c, R, t, g, Dt, Ct, rng = scene(200 + seed, n=3)
    r = rng.normal(size=(c.height, c.width, 3))
    out = O.render(g, c, R, t, Dt, Ct)
    grads, _ = O.backward(g, c, R, t, Dt, out["Cstar"], out["WG"], r)
    g64 = {k: (np.asarray(v, np.float64).copy() if isinstance(v, np.ndarray) else v) for k, v in g.items()}
    base_ind = RI.render_allpairs(RI.to_torch_params(g64), cam_tuple(c), R, t, Dt, Ct)[2]
    checked = 0
    for k in GROUPS:
        arr = g64[k]
        flat = arr.reshape(-1)
        for j in range(flat.size):
            th = flat[j]
            h = 1e-5 * max(1.0, abs(th))
            vals = []
            same = True
            for sgn in (1, -1):
                flat[j] = th + sgn * h
                ind = RI.render_allpairs(RI.to_torch_params(g64), cam_tuple(c), R, t, Dt, Ct)[2]
                same &= bool(torch.equal(ind, base_ind))
                o2 = O.render(g64, c, R, t, Dt, Ct)
                vals.append(float((o2["Cstar"] * r).sum()))
            flat[j] = th
            if not same:
                continue
            fd = (vals[0] - vals[1]) / (2 * h)
            an = grads[k].reshape(-1)[j]
            # 1e-5 relative, plus the fp64 rounding floor of the summed functional / (2h)
            assert abs(fd - an) <= 1e-5 * abs(an) + 1e-8, (k, j, fd, an)
            checked += 1
    assert checked > 100


def test_zero_upstream_gives_zero_gradient():
    """zero upstream gradient -> all parameter gradients zero."""
    c, R, t, g, Dt, Ct, _ = scene(300)
    out = O.render(g, c, R, t, Dt, Ct)
    grads, _ = O.backward(g, c, R, t, Dt, out["Cstar"], out["WG"], np.zeros((c.height, c.width, 3)))
    for v in grads.values():
        assert np.all(v == 0)


def test_single_gaussian_opacity_gradient_closed_form():
    """At its centre pixel a lone Gaussian has dC*/do_raw = sigma(1-sigma)(c - C*)/(1+W_G)
    (d alpha/d sigma = 1 there); with upstream = indicator of that pixel's red channel."""
    c = small_cam(33, 25, 30.0, cx=16.0, cy=12.0)
    g = one_gaussian((0, 0, 1.0), (0.01, 0.01, 0.01), o=0.3, sh0=(0.7, 0.0, 0.0))
    Ct = np.full((c.height, c.width, 3), 0.2)
    Dt = np.zeros((c.height, c.width))
    out = O.render(g, c, np.eye(3), np.zeros(3), Dt, Ct)
    G = np.zeros((c.height, c.width, 3))
    G[12, 16, 0] = 1.0
    grads, _ = O.backward(g, c, np.eye(3), np.zeros(3), Dt, out["Cstar"], out["WG"], G)
    o = np.float64(g["opacity_raw"][0])  # the stored fp32 values
    sig = 1 / (1 + np.exp(-o))
    col = 0.28209479177387814 * np.float64(g["sh"][0, 0]) + 0.5
    W = out["WG"][12, 16]
    expect = sig * (1 - sig) * (col - out["Cstar"][12, 16, 0]) / (1 + W)
    assert abs(grads["opacity_raw"][0] - expect) < 1e-14
