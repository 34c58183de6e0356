"""Pins of the oracle's tile lists (north_star "tile binning with a (tile, depth) key sort";
DESIGN.md §4.3) and of its Adam (torch formula: "Libtorch", learning rates App. C
P:455; reading R-ADAM)."""
import numpy as np
import pytest
import torch

import oracle as O
from gps_synth import random_gaussians
from tests import refimpl as RI


def scene(seed, n=300, w=70, h=45):
    rng = np.random.default_rng(seed)
    c = O.Camera(50.0, 50.0, (w - 1) / 2 + 0.3, (h - 1) / 2 - 0.2, w, h)
    R = RI.random_rotation(rng)
    t = rng.uniform(-0.1, 0.1, 3).astype(np.float32)
    ctr = R.astype(np.float64) @ np.array([0, 0, 1.2]) + t
    g = random_gaussians(n, 1, rng, center=ctr, spread=0.6, scale=(0.002, 0.05))
    return c, R, t, g


@pytest.mark.parametrize("tile", [8, 16])
@pytest.mark.parametrize("seed", [0, 1])
def test_tile_lists_brute_force(seed, tile):
    """Brute force over tile x Gaussian with explicit pixel sets: Gaussian i is in List(T) iff
    its P32 rect and T share a pixel; each list ascends by (depth bits, index); ranges partition
    [0, K) in tile order; K = sum over Gaussians of touched tiles."""
    c, R, t, g = scene(seed)
    rect, depth, culled = O.project_p32(g, c, R, t, O.RenderCfg())
    values, ranges = O.tile_lists(rect, depth, culled, c.width, c.height, tile)
    tx = -(-c.width // tile)
    ty = -(-c.height // tile)
    assert ranges.shape == (tx * ty, 2)
    assert ranges[0, 0] == 0 and ranges[-1, 1] == len(values)
    assert np.all(ranges[1:, 0] == ranges[:-1, 1])
    for T in range(tx * ty):
        x0, y0 = (T % tx) * tile, (T // tx) * tile
        mask = np.zeros((c.height, c.width), bool)
        mask[y0:y0 + tile, x0:x0 + tile] = True
        expect = []
        for i in range(len(depth)):
            if culled[i]:
                continue
            r = np.zeros_like(mask)
            r[rect[i, 1]:rect[i, 3] + 1, rect[i, 0]:rect[i, 2] + 1] = True
            if (r & mask).any():
                expect.append((depth[i].view(np.uint32), i))
        expect.sort()
        got = values[ranges[T, 0]:ranges[T, 1]]
        assert list(got) == [i for _, i in expect]
    assert (culled == 0).sum() > 100


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_p32_rect_covers_footprint_and_depth_matches(seed):
    """The P32 rect (tile membership) contains every pixel where the Gaussian is in (Eqs. 1-3
    with the 3-sigma reading R-FOOT, computed in fp64 by the independent torch forward), and
    the P32 depth/cull agree with fp64 (relative 1e-6)."""
    c, R, t, g = scene(seed, n=200)
    rect, depth, culled = O.project_p32(g, c, R, t, O.RenderCfg())
    Dt = np.zeros((c.height, c.width))
    Ct = np.zeros((c.height, c.width, 3))
    _, _, ind = RI.render_allpairs(RI.to_torch_params(g), (c.fx, c.fy, c.cx, c.cy, c.width, c.height),
                                   R, t, Dt, Ct)
    ind = ind.numpy().reshape(len(depth), c.height, c.width)
    pr = RI.project(RI.to_torch_params(g), (c.fx, c.fy, c.cx, c.cy, c.width, c.height), R, t)
    z64 = pr["depth"].numpy()
    assert np.max(np.abs(depth - z64) / np.abs(z64)) < 1e-6
    for i in range(len(depth)):
        ys, xs = np.nonzero(ind[i])
        if len(xs) == 0:
            continue
        assert culled[i] == 0
        assert xs.min() >= rect[i, 0] and xs.max() <= rect[i, 2]
        assert ys.min() >= rect[i, 1] and ys.max() <= rect[i, 3]
    # the rect is tight: the 3-sigma ellipse box, rounded outward by < 1 px
    s2 = pr["S2"].numpy()
    ok = culled == 0
    rx = 3 * np.sqrt(s2[ok, 0, 0])
    px = pr["p_hat"].numpy()[ok, 0]
    inner = (rect[ok, 0] > 0) & (rect[ok, 2] < c.width - 1)
    w = (rect[ok, 2] - rect[ok, 0])[inner]
    assert np.all(w <= np.ceil(px + rx)[inner] - np.floor(px - rx)[inner])
    assert np.all(w >= 2 * rx[inner] - 1e-3)


# ---------------------------------------------------------------------------------------------
def params_like(rng, n=7, deg=2):
    g = random_gaussians(n, deg, rng)
    return {k: np.asarray(v, np.float64) for k, v in g.items() if k != "sh_degree"}


def test_adam_matches_torch_optim():
    """O10: five dense steps of the oracle Adam equal torch.optim.Adam (fp64, eps=1e-15, per-
    group learning rates; sh0 and the other SH coefficients as separate groups) to 1e-12."""
    rng = np.random.default_rng(0)
    cfg = O.AdamCfg()
    p = params_like(rng)
    n = p["xyz"].shape[0]
    m = {k: np.zeros_like(v) for k, v in p.items()}
    v = {k: np.zeros_like(v) for k, v in p.items()}
    tp = {k: torch.tensor(val.copy(), requires_grad=True) for k, val in p.items()}
    sh = tp.pop("sh")
    sh0 = torch.tensor(p["sh"].reshape(n, -1, 3)[:, :1].copy(), requires_grad=True)
    shr = torch.tensor(p["sh"].reshape(n, -1, 3)[:, 1:].copy(), requires_grad=True)
    lr = O.lr_groups(cfg)
    opt = torch.optim.Adam([{"params": [tp["xyz"]], "lr": lr["xyz"]},
                            {"params": [tp["log_scale"]], "lr": lr["log_scale"]},
                            {"params": [tp["rot"]], "lr": lr["rot"]},
                            {"params": [tp["opacity_raw"]], "lr": lr["opacity_raw"]},
                            {"params": [sh0], "lr": cfg.lr_sh0},
                            {"params": [shr], "lr": cfg.lr_shrest}],
                           betas=(cfg.beta1, cfg.beta2), eps=cfg.eps)
    for step in range(5):
        g = {k: rng.normal(size=val.shape) * 10.0 ** rng.uniform(-8, 0) for k, val in p.items()}
        if step == 2:
            g["xyz"][0] = 0.0
        p, m, v = O.adam_step(p, m, v, g, step, cfg)
        for k in ("xyz", "log_scale", "rot", "opacity_raw"):
            tp[k].grad = torch.tensor(g[k])
        gs = g["sh"].reshape(n, -1, 3)
        sh0.grad = torch.tensor(gs[:, :1].copy())
        shr.grad = torch.tensor(gs[:, 1:].copy())
        opt.step()
        for k in ("xyz", "log_scale", "rot", "opacity_raw"):
            assert np.max(np.abs(p[k] - tp[k].detach().numpy()) / (np.abs(p[k]) + 1e-300)) < 1e-12, k
        ref_sh = torch.cat([sh0, shr], dim=1).detach().numpy()
        assert np.max(np.abs(p["sh"].reshape(n, -1, 3) - ref_sh)) < 1e-12


def test_adam_first_step_closed_form_and_zero_gradient():
    """First step: p1 = p0 - lr g/(|g| + eps) (bias corrections cancel); a zero gradient at
    t = 1 leaves the parameter unchanged; a constant gradient gives steps -> lr
    (S:335)."""
    cfg = O.AdamCfg()
    p0 = np.array([0.5, -1.0, 2.0])
    g = np.array([3e-7, -2.0, 0.0])
    p1, m, v = O.adam_update(p0, np.zeros(3), np.zeros(3), g, 0.01, 1, 0.9, 0.999, 1e-15)
    assert np.allclose(p1, p0 - 0.01 * g / (np.abs(g) + 1e-15), rtol=0, atol=1e-15)
    assert p1[2] == p0[2]
    p = p0.copy()
    m = np.zeros(3)
    v = np.zeros(3)
    for t in range(1, 200):
        pn, m, v = O.adam_update(p, m, v, np.array([1.0, 1.0, 1.0]), 0.01, t, 0.9, 0.999, 1e-15)
        step = p - pn
        p = pn
    assert np.allclose(step, 0.01, rtol=1e-6)
