"""GPU parity of gps_render / gps_refine_step / gps_adam_step against the CPU oracle
(SURVEY §8(c) O5-O10).  Inputs are seeded (gps_synth): analytic-scene D_t/C_t stand-ins, so the
render stage is compared without consuming any CUDA output.

Bars: tile lists bit-exact (both sides bin the prescribed-fp32 projection fields);
C* within 1e-3 absolute and W_G within 1e-3 relative on unambiguous pixels; loss within 1e-5
relative; raw-parameter gradients within 1e-3 relative with the floor tau = 1e-3 max|g| per block
(Gaussians touching an ambiguous decision excluded and counted); Adam within 1e-6 relative on
identical gradients.  PAPER.md Eqs. 1-4, Eq. 7."""
import numpy as np
import pytest
import torch

import gps_synth as S
import oracle as O
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu

GROUPS = ("xyz", "log_scale", "rot", "opacity_raw", "sh")


def setup(cfg_name="cfg1", start=0, n=None):
    import paper_2509_11574_b200 as G
    cfg = S.get_config(cfg_name)
    fr = H.frames(cfg, 1, start=start)[0]
    gd = S.make_gaussians(cfg, n=n, frames=[fr] if cfg_name == "cfg1" else None)
    Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=start)
    tgt = S.target_rgba(cfg, fr)
    gcam, ocam = H.cams(cfg)
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=tgt.cuda().contiguous())
    return G, cfg, fr, gd, Dt, Ct, tgt.numpy(), gcam, ocam, dev


def gpu_render(G, gd, gcam, fr, dev, tile=16, precull=0, target=True):
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile=tile, tile_depth_precull=precull))
    Cs, W, loss = ras.render(g, gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"] if target else None)
    torch.cuda.synchronize()
    return ras, Cs.cpu().numpy(), W.cpu().numpy(), (loss.item() if loss is not None else None)


def check_forward(out, Cs, W):
    """Pair membership is decided bit-identically on both sides, so every
    pixel is compared: C* within 1e-3 absolute, W_G within 1e-3 relative."""
    assert np.max(np.abs(Cs - out["Cstar"])) <= 1e-3
    assert np.all(np.abs(W - out["WG"]) <= 1e-3 * out["WG"] + 1e-6)
    assert np.all((W > 0) == (out["WG"] > 0))
    assert out["WG"].max() > 0.5


@pytest.mark.parametrize("tile", [16, 8])
def test_render_cfg1_matches_oracle_and_lists_bit_exact(tile):
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    ras, Cs, W, loss = gpu_render(G, gd, gcam, fr, dev, tile=tile, precull=0)
    out = O.render(gd, ocam, fr.R, fr.t, Dt, Ct)
    check_forward(out, Cs, W)
    ol, _, cnt, _ = O.l1_loss(out["Cstar"], out["WG"], Dt, tgt)
    assert abs(loss - ol) <= 1e-5 * ol
    # tile lists: bit-exact against the oracle's binning of its own P32 projection
    rect, depth, culled = O.project_p32(gd, ocam, fr.R, fr.t, O.RenderCfg())
    ov, orng = O.tile_lists(rect, depth, culled, cfg.width, cfg.height, tile)
    gv, grng = ras.lists()
    assert np.array_equal(grng, orng)
    assert np.array_equal(gv, ov)
    st = ras.stats()
    assert st["pairs"] == len(ov) and st["n_visible"] == int((culled == 0).sum()) and st["status"] == "GPS_OK"


def test_precull_and_early_exit_do_not_change_the_image():
    """Early termination at the SDF depth and the tile pre-cull skip only entries that add exact
    zeros (lists are depth-sorted), so the image is bitwise unchanged; the
    truncated lists are prefixes of the full ones.  Rendering is deterministic."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    ras0, C0, W0, l0 = gpu_render(G, gd, gcam, fr, dev, precull=0)
    v0, r0 = ras0.lists()
    ras1, C1, W1, l1 = gpu_render(G, gd, gcam, fr, dev, precull=1)
    v1, r1 = ras1.lists()
    assert np.array_equal(C0, C1) and np.array_equal(W0, W1) and l0 == l1
    assert np.array_equal(r0[:, 0], r1[:, 0]) and np.all(r1[:, 1] <= r0[:, 1])
    for t in range(len(r0)):
        assert np.array_equal(v1[r1[t, 0]:r1[t, 1]], v0[r0[t, 0]:r0[t, 0] + (r1[t, 1] - r1[t, 0])])
    _, C2, W2, l2 = gpu_render(G, gd, gcam, fr, dev, precull=1)
    assert np.array_equal(C1, C2) and np.array_equal(W1, W2) and l1 == l2


def test_zero_gaussians_compose_identity():
    """AC1: with no Gaussians C* = C_t bitwise and W_G = 0."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    g0 = {k: (v[:0] if isinstance(v, np.ndarray) else v) for k, v in gd.items()}
    _, Cs, W, _ = gpu_render(G, g0, gcam, fr, dev)
    assert np.array_equal(Cs, Ct) and np.all(W == 0)


@pytest.mark.slow
def test_render_full_size_cfg4():
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup("cfg4", start=300)
    ras, Cs, W, loss = gpu_render(G, gd, gcam, fr, dev, precull=1)
    out = O.render(gd, ocam, fr.R, fr.t, Dt, Ct)
    check_forward(out, Cs, W)
    ol = O.l1_loss(out["Cstar"], out["WG"], Dt, tgt)[0]
    assert abs(loss - ol) <= 1e-5 * ol


# ---------------------------------------------------------------------------------------------
def oracle_grads(gd, ocam, R, t, Dt, Ct, tgt, with_sens=False):
    out = O.render(gd, ocam, R, t, Dt, Ct)
    loss, G, cnt, samb = O.l1_loss(out["Cstar"], out["WG"], Dt, tgt)
    # only sign(C* - C_k) ties (|C* - C_k| < 1e-5) can legitimately differ: membership is exact
    grads, gamb = O.backward(gd, ocam, R, t, Dt, out["Cstar"], out["WG"], G, pix_amb=samb)
    if with_sens:  # full-size images: the fp32 conditioning allowance of compare_grads
        return loss, grads, gamb, grad_sensitivity(gd, ocam, R, t, Dt, out["Cstar"], out["WG"], G, samb)
    return loss, grads, gamb


def grad_sensitivity(gd, ocam, R, t, Dt, Cstar, WG, G, pix_amb, rel=5e-7, prel=2e-7, seed=0):
    """How much the oracle's own gradient moves under fp32-rounding-level perturbations of what
    the CUDA path computes in fp32: C* scaled by (1 +- 5e-7) (8 fp32 ulps, coherent over the
    image), and every Gaussian position scaled by (1 + 2e-7 r), r = +-1 per Gaussian (the fp32
    projection's error of p_hat).  Elementwise max of |change|: the scale of the legitimate fp32
    error of a gradient that sums cancelling terms (dL/dalpha ~ c - C* small, or symmetric
    footprints cancelling dL/dp_hat; R-GRAD)."""
    rng = np.random.default_rng(seed)
    base, _ = O.backward(gd, ocam, R, t, Dt, Cstar, WG, G, pix_amb=pix_amb)
    out = {k: np.zeros_like(v) for k, v in base.items()}
    C = np.asarray(Cstar, np.float64)
    gp = dict(gd, xyz=(np.asarray(gd["xyz"], np.float64)
                       * (1.0 + prel * rng.choice([-1.0, 1.0], size=(len(gd["xyz"]), 1)))))
    for args in ((gd, C * (1.0 + rel)), (gd, C * (1.0 - rel)), (gp, C)):
        g2, _ = O.backward(args[0], ocam, R, t, Dt, args[1], WG, G, pix_amb=pix_amb)
        for k in GROUPS:
            out[k] = np.maximum(out[k], np.abs(g2[k] - base[k]))
    return out


def compare_grads(gg, ref, gamb, min_checked=50, sens=None):
    """O9: |g_gpu - g_ref| <= 1e-3 max(|g_ref|, tau), tau = 1e-3 max|g_ref| per parameter block.
    With `sens` (grad_sensitivity), a value may instead be within 4x the gradient's sensitivity
    to fp32 rounding of C* (an ill-conditioned dL/dalpha); such values are counted and must be
    <= 1e-3 of those compared."""
    keep = ~gamb
    assert keep.sum() >= min_checked
    n_sens = n_tot = 0
    for k in GROUPS:
        a = gg[k].reshape(len(keep), -1)[keep]
        b = ref[k].reshape(len(keep), -1)[keep]
        tau = 1e-3 * np.max(np.abs(b))
        assert tau > 0, k
        err = np.abs(a - b) / np.maximum(np.abs(b), tau)
        bad = err > 1e-3
        if sens is not None:
            sk = sens[k].reshape(len(keep), -1)[keep]
            explained = bad & (np.abs(a - b) <= 4.0 * sk)
            n_sens += int(explained.sum())
            bad &= ~explained
        n_tot += err.size
        assert not bad.any(), (k, float(err[bad].max()), int(bad.sum()))
    if sens is not None:
        print(f"gradients: {n_tot} values compared, {n_sens} within 4x their fp32 C* sensitivity only")
        assert n_sens <= max(2, 1e-3 * n_tot)


def test_refine_gradients_and_adam_cfg1():
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    g = G.Gaussians.from_dict(gd)
    p0 = g.to_numpy()
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
    view = G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    loss = ras.refine_step(g, st, [view], grad_out=gout).item()
    assert st.step == 1
    oloss, ref, gamb = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt)
    assert abs(loss - oloss) <= 1e-5 * oloss
    gg = gout.to_numpy()
    compare_grads(gg, ref, gamb)
    # Adam step 1: p1 = p0 - lr g/(|g| + eps): equal to the oracle's update of the oracle gradient
    # wherever |g| is above the per-block floor (sign-like below it: may differ by 2 lr)
    m0 = {k: np.zeros_like(np.asarray(p0[k], np.float64)) for k in GROUPS}
    P1, _, _ = O.adam_step(p0, m0, m0, ref, 0)
    p1 = g.to_numpy()
    for k in GROUPS:
        b = ref[k].reshape(len(gamb), -1)
        sel = (np.abs(b) > 1e-2 * np.max(np.abs(b))) & ~gamb[:, None]
        a1 = p1[k].reshape(len(gamb), -1)[sel]
        e1 = P1[k].reshape(len(gamb), -1)[sel]
        assert np.max(np.abs(a1 - e1)) <= 1e-6 * np.max(np.abs(e1)) + 1e-7, k


def test_adam_step_identical_gradients():
    """O10: given identical gradients the device Adam equals the oracle's (3 steps)."""
    import paper_2509_11574_b200 as G
    rng = np.random.default_rng(3)
    gd = S.random_gaussians(777, 3, rng)
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    P = {k: np.asarray(gd[k], np.float64) for k in GROUPS}
    M = {k: np.zeros_like(v) for k, v in P.items()}
    V = {k: np.zeros_like(v) for k, v in P.items()}
    for step in range(3):
        gr = {k: (rng.normal(size=np.shape(gd[k])) * 10.0 ** rng.uniform(-6, 0)).astype(np.float32) for k in GROUPS}
        G.adam_step(g, st, G.Gaussians.from_dict({**gr, "sh_degree": 3}))
        P, M, V = O.adam_step(P, M, V, {k: np.asarray(v, np.float64) for k, v in gr.items()}, step)
    torch.cuda.synchronize()
    got = g.to_numpy()
    lr = {"xyz": 1.6e-4, "log_scale": 5e-3, "rot": 1e-3, "opacity_raw": 5e-2, "sh": 2.5e-3}
    for k in GROUPS:
        # 1e-6 relative, plus fp32 rounding of the three updates (absolute, ~ lr)
        Pk = np.asarray(P[k]).reshape(got[k].shape)
        err = np.abs(got[k] - Pk) - 1e-6 * np.abs(Pk)
        assert err.max() <= 1e-6 * 3 * lr[k], (k, err.max())
    assert st.step == 3


def test_refine_two_views_sums_gradients():
    """n_views = 2 (SPEC's all-views variant): gradients and losses of the views add."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    R2 = np.asarray(fr.R, np.float32)
    t2 = (np.asarray(fr.t) + np.array([0.004, -0.003, 0.0])).astype(np.float32)
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(), n_views=2)
    views = [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"]),
             G.View(gcam, R2, t2, dev["Dt"], dev["Ct"], dev["tgt"])]
    loss = ras.refine_step(g, st, views, grad_out=gout).item()
    l1, r1, a1 = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt)
    l2, r2, a2 = oracle_grads(gd, ocam, R2, t2, Dt, Ct, tgt)
    assert abs(loss - (l1 + l2)) <= 1e-5 * (l1 + l2)
    compare_grads(gout.to_numpy(), {k: r1[k] + r2[k] for k in GROUPS}, a1 | a2)


def test_refinement_reduces_the_loss():
    """20 iterations on one view lower the L1 loss (SPEC S:336 monotone toy fit)."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
    view = G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    losses = [ras.refine_step(g, st, [view]).item() for _ in range(20)]
    assert losses[-1] < losses[0] * 0.98


@pytest.mark.slow
def test_refine_gradients_full_size_cfg4():
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup("cfg4", start=300)
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
    view = G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    loss = ras.refine_step(g, st, [view], grad_out=gout).item()
    oloss, ref, gamb, sens = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt, with_sens=True)
    assert abs(loss - oloss) <= 1e-5 * oloss
    got = gout.to_numpy()
    import os
    if os.path.isdir("gpurun_out"):  # diagnostics for offline analysis
        np.savez_compressed("gpurun_out/cfg4_grads.npz", **{k: np.asarray(got[k], np.float32)[:, :12]
                                                            if k == "sh" else got[k] for k in GROUPS})
    compare_grads(got, ref, gamb, min_checked=10000, sens=sens)


@pytest.mark.parametrize("deg", [0, 1, 2])
def test_render_and_gradients_other_sh_degrees(deg):
    """SH degrees 0-2 (P = 14, 23, 38 floats/Gaussian): render and raw gradients match."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    rng = np.random.default_rng(10 + deg)
    nc = (deg + 1) ** 2
    gd = dict(gd, sh_degree=deg, sh=np.ascontiguousarray(gd["sh"].reshape(len(gd["xyz"]), 16, 3)[:, :nc].reshape(-1, 3 * nc)))
    _, Cs, W, loss = gpu_render(G, gd, gcam, fr, dev)
    out = O.render(gd, ocam, fr.R, fr.t, Dt, Ct)
    check_forward(out, Cs, W)
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
    ras.refine_step(g, st, [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt)
    compare_grads(gout.to_numpy(), ref, gamb)


@pytest.mark.parametrize("tile,precull", [(8, 1), (16, 1), (8, 0)])
def test_refine_gradients_tile_variants(tile, precull):
    """The tile size and the tile pre-cull are accelerators: gradients equal the oracle's."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile=tile, tile_depth_precull=precull))
    ras.refine_step(g, st, [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt)
    compare_grads(gout.to_numpy(), ref, gamb)


def test_large_gaussians_span_many_tiles():
    """Gaussians whose rect spans more than 4 tiles take the cursor path of the binning; lists
    stay bit-exact and gradients match (wide random scales on a 160x120 view)."""
    import paper_2509_11574_b200 as G
    rng = np.random.default_rng(5)
    c = O.Camera(120.0, 120.0, 79.5, 59.5, 160, 120)
    gcam = G.Camera(120.0, 120.0, 79.5, 59.5, 160, 120)
    R, t = np.eye(3, dtype=np.float32), np.zeros(3, np.float32)
    gd = S.random_gaussians(300, 1, rng, center=(0, 0, 1.0), spread=0.4, scale=(0.005, 0.12))
    Dt = rng.uniform(1.1, 1.5, (120, 160)).astype(np.float32)
    Ct = rng.random((120, 160, 3)).astype(np.float32)
    tgt = rng.integers(0, 256, (120, 160, 4)).astype(np.uint8)
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=torch.from_numpy(tgt).cuda())
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile_depth_precull=0))
    Cs, W, loss = ras.render(g, gcam, R, t, dev["Dt"], dev["Ct"], dev["tgt"])
    rect, depth, culled = O.project_p32(gd, c, R, t, O.RenderCfg())
    spans = [((r[2] // 16) - (r[0] // 16) + 1) * ((r[3] // 16) - (r[1] // 16) + 1) for r, cu in zip(rect, culled) if not cu]
    assert max(spans) > 4 and min(spans) <= 4
    ov, orng = O.tile_lists(rect, depth, culled, 160, 120, 16)
    gv, grng = ras.lists()
    assert np.array_equal(grng, orng) and np.array_equal(gv, ov)
    out = O.render(gd, c, R, t, Dt, Ct)
    check_forward(out, Cs.cpu().numpy(), W.cpu().numpy())
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras.refine_step(g, st, [G.View(gcam, R, t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, c, R, t, Dt, Ct, tgt)
    compare_grads(gout.to_numpy(), ref, gamb, min_checked=20)


def test_two_pixel_blend_is_bitwise_the_one_pixel_blend(tmp_path):
    """k_sort_blend16x2 (default for 16x16 tiles: per-warp walk, packed f32x2) processes, per
    pixel, the same entries in the same order with the same roundings as k_sort_blend<16>
    (GPS_BLEND_1PX=1) and as its CTA-staged scalar form (GPS_BLEND_STAGED=1; both read once per
    process): C*, W_G and the loss are bitwise equal.  cfg2-sized frame, 50k Gaussians, sorted and sort-free."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import gps_synth as S, paper_2509_11574_b200 as G
cfg = S.get_config("cfg2")
fr = S.make_frames(cfg, 1, start=5)[0]
gd = S.make_gaussians(cfg, n=50000)
Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=5)
cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
out = {}
for sf in (0, 1):
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, cam, G.RenderConfig(sort_free=sf))
    C, W, l = ras.render(g, cam, fr.R, fr.t, torch.from_numpy(Dt).cuda(), torch.from_numpy(Ct).cuda(),
                         fr.rgba.cuda().contiguous())
    torch.cuda.synchronize()
    out[f"C{sf}"], out[f"W{sf}"], out[f"l{sf}"] = C.cpu().numpy(), W.cpu().numpy(), np.array([l.item()])
np.savez(sys.argv[2], **out)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for name, env in (("two", {}), ("one", {"GPS_BLEND_1PX": "1"}), ("staged", {"GPS_BLEND_STAGED": "1"})):
        path = str(tmp_path / f"{name}.npz")
        e = {k: v for k, v in os.environ.items() if k not in ("GPS_BLEND_1PX", "GPS_BLEND_STAGED")}
        e.update(env)
        subprocess.run([sys.executable, "-c", code, root, path], check=True, env=e, timeout=600)
        res[name] = np.load(path)
    for k in ("C0", "W0", "l0"):
        assert np.array_equal(res["two"][k], res["one"][k]), k
        assert np.array_equal(res["two"][k], res["staged"][k]), k  # warp walk + f32x2 vs CTA-staged
    # sort-free: the bucket order comes from atomics, so only agreement to rounding is expected
    assert np.max(np.abs(res["two"]["C1"] - res["one"]["C1"])) <= 1e-5


def test_pair_counters_accepted_matches_an_independent_count():
    """gps_debug_render_counts_sync's accepted pairs A equal the number of
    (pixel, Gaussian) pairs passing the exact membership of DESIGN.md §4.3 and the Eq. 1 depth
    indicator, counted here from the oracle's P32 fields (fp32, FMA emulated through exact fp64
    products: boundary double-rounding allowed for, 1e-4); the evaluated pairs E bound A."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2")
    fr = H.frames(cfg, 1, start=3)[0]
    gd = S.make_gaussians(cfg, n=20000)
    Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=3)
    gcam, ocam = H.cams(cfg)
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile_depth_precull=1))
    E, A = ras.pair_counts(g, gcam, fr.R, fr.t, torch.from_numpy(Dt).cuda(), torch.from_numpy(Ct).cuda())
    rect, depth, culled, fl = O.project_p32(gd, ocam, fr.R, fr.t, O.RenderCfg(), fields=True)
    f32 = np.float32
    L = f32(-np.log(np.float64(f32(1.0 / 255))))
    eps = f32(0.02)
    count = 0
    for i in np.flatnonzero(culled == 0):
        x0, y0, x1, y1 = rect[i]
        px, py, a, b, c, lns = fl[i]
        qmax = min(f32(9.0), f32(f32(2.0) * f32(L + lns)))
        xs = np.arange(x0, x1 + 1, dtype=f32)
        ys = np.arange(y0, y1 + 1, dtype=f32)
        dx = (xs[None, :] - px).astype(f32)
        dy = (ys[:, None] - py).astype(f32)
        b2 = f32(f32(2.0) * b)
        inner = ((b2 * dx).astype(f32).astype(np.float64) * dy + ((c * dy).astype(f32) * dy).astype(f32)).astype(f32)
        q = ((a * dx).astype(f32).astype(np.float64) * dx + inner).astype(f32)
        D = Dt[y0:y1 + 1, x0:x1 + 1]
        ok = (q <= qmax) & ((D == 0) | (depth[i] < (D + eps).astype(f32)))
        count += int(ok.sum())
    assert A > 1000 and E >= A
    assert abs(A - count) <= 1e-4 * count


def test_tile_lists_with_equal_depths_bit_exact():
    """Entries sharing a depth (duplicated Gaussian centres) are ordered by index: the 16x16
    blend's 32-bit depth rank detects the tie and re-ranks the tile on the (depth, index) keys;
    lists and image stay bit-exact / within the bars against the oracle."""
    import paper_2509_11574_b200 as G
    G_, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    gd = {k: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v) for k, v in gd.items()}
    n = len(gd["opacity_raw"])
    rng = np.random.default_rng(9)
    src = rng.choice(n, size=n // 4, replace=False)
    dst = rng.choice(np.setdiff1d(np.arange(n), src), size=n // 4, replace=False)
    gd["xyz"].reshape(n, 3)[dst] = gd["xyz"].reshape(n, 3)[src]  # same centre -> same depth bits
    ras, Cs, W, loss = gpu_render(G, gd, gcam, fr, dev, tile=16, precull=0)
    rect, depth, culled = O.project_p32(gd, ocam, fr.R, fr.t, O.RenderCfg())
    vis = culled == 0
    assert len(np.unique(depth[vis])) < vis.sum()  # ties are present
    ov, orng = O.tile_lists(rect, depth, culled, cfg.width, cfg.height, 16)
    gv, grng = ras.lists()
    assert np.array_equal(grng, orng) and np.array_equal(gv, ov)
    check_forward(O.render(gd, ocam, fr.R, fr.t, Dt, Ct), Cs, W)


@pytest.mark.parametrize("deg,n", [(3, 50001), (1, 1001)])
def test_fused_chain_adam_matches_the_unfused_pair(deg, n, monkeypatch):
    """k_chain_adam (single-view refine steps) applies the same chain rule and the same Adam
    arithmetic as k_chain + k_adam (GPS_UNFUSED_ADAM=1, read per call).  The backward's 2D
    gradient totals arrive by fp32 atomics (order-dependent in the last bits), so two runs agree
    to rounding, not bitwise: raw gradients and moments within 1e-4 relative (plus 1e-6 of the
    group's largest), parameters within 2 lr (Adam's first step is ~lr sign(g)).  n not a multiple
    of the 128-Gaussian chunk, 3n not a multiple of 4 (ragged chunk and float4 units)."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2")
    fr = H.frames(cfg, 1, start=5)[0]
    gd = S.make_gaussians(cfg, n=n, sh_degree=deg)
    Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=5)
    tgt = S.target_rgba(cfg, fr).cuda().contiguous()
    gcam, _ = H.cams(cfg)
    view = G.View(gcam, fr.R, fr.t, torch.from_numpy(Dt).cuda(), torch.from_numpy(Ct).cuda(), tgt)
    res = {}
    for mode in ("fused", "unfused"):
        if mode == "unfused":
            monkeypatch.setenv("GPS_UNFUSED_ADAM", "1")
        else:
            monkeypatch.delenv("GPS_UNFUSED_ADAM", raising=False)
        g = G.Gaussians.from_dict(gd)
        st = G.AdamState(g)
        gout = g.zeros_like()
        ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
        loss = ras.refine_step(g, st, [view], grad_out=gout).item()
        torch.cuda.synchronize()
        res[mode] = (loss, g.to_numpy(), st.m.to_numpy(), st.v.to_numpy(), gout.to_numpy())
    lr = {"xyz": 1.6e-4, "log_scale": 5e-3, "rot": 1e-3, "opacity_raw": 5e-2, "sh": 2.5e-3}
    fu = res["unfused"]
    for fl in (res["fused"],):
        assert fl[0] == fu[0]  # the forward is bit-reproducible
        for k in GROUPS:
            for j, (a, b) in enumerate(((fl[4][k], fu[4][k]), (fl[2][k], fu[2][k]), (fl[3][k], fu[3][k]))):
                a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
                assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b) + 1e-6 * np.abs(b).max()), k
                # the gradient's support is exact; m and v may underflow (denormal v) differently
                assert j > 0 or (np.count_nonzero(b) > 0 and np.array_equal(a != 0, b != 0)), k
            assert np.max(np.abs(np.asarray(fl[1][k], np.float64) - fu[1][k])) <= 2 * lr[k], k


def _round_views(G, cfg, frs, window):
    """Views of frames frs through a (x0, y0, w, h) window of the camera (a crop: same rays)."""
    x0, y0, w, h = window
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx - x0, cfg.cy - y0, w, h)
    views = []
    for i, fr in enumerate(frs):
        Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=11 + i)
        tgt = S.target_rgba(cfg, fr)
        crop = (slice(y0, y0 + h), slice(x0, x0 + w))
        views.append(G.View(cam, fr.R, fr.t, torch.from_numpy(np.ascontiguousarray(Dt[crop])).cuda(),
                            torch.from_numpy(np.ascontiguousarray(Ct[crop])).cuda(),
                            tgt[crop].contiguous().cuda()))
    return cam, views


def _run_round(G, gd, cam, views, plan, mode, stream):
    """plan: list of rounds, each a list of per-iteration view-index lists."""
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    ras = G.Rasterizer(g.n, cam, G.RenderConfig(), n_views=max(len(it) for r in plan for it in r))
    losses = []
    stream.wait_stream(torch.cuda.current_stream())  # the parameters and moments are initialised
    with torch.cuda.stream(stream):
        for order in plan:
            if mode.startswith("steps"):
                for vi in order:
                    ras.refine_step(g, st, [views[j] for j in vi], stream=stream)
            else:
                ras.refine_round(g, st, views, order, graph=(mode == "graph"), stream=stream)
            # no synchronisation between rounds: a graph round may be updated while an earlier
            # one is still in flight
            losses.append(ras.loss.clone())
    torch.cuda.synchronize()
    return st.step, [x.item() for x in losses], g.to_numpy(), st.m.to_numpy(), st.v.to_numpy()


def test_refine_round_graph_is_bitwise_the_refine_steps():
    """gps_refine_round (one call per round; use_graph: the round captured and replayed as one
    CUDA graph, updated in place for the next round of the same shape, re-instantiated for a
    round of another length) launches the same kernels in the same order as the per-iteration
    gps_refine_step calls.  On a single 16x16 tile every Gaussian's 2D gradient arrives in one
    atomic per view (deterministic), so the three schedules are compared bitwise: parameters,
    moments, step counts and each round's last loss."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2")
    frs = H.frames(cfg, 3, start=4)
    cam, views = _round_views(G, cfg, frs, (312, 232, 16, 16))
    gd = S.make_gaussians(cfg, n=3000, sh_degree=3)
    plan = [[[i % 3] for i in range(7)], [[(i + 1) % 3] for i in range(7)], [[2], [0], [1]],
            [[0], [0], [2]], [[1], [2], [0]], [[i % 3] for i in range(7)], [[2], [2], [1]]]
    s = torch.cuda.Stream()
    res = {m: _run_round(G, gd, cam, views, plan, m, s) for m in ("steps", "steps2", "direct", "graph")}
    ref = res["steps"]
    assert ref[0] == 7 + 7 + 3 + 3 + 3 + 7 + 3 and all(l > 0 for l in ref[1])
    for m in ("steps2", "direct", "graph"):  # steps2: the schedule is reproducible at all
        r = res[m]
        assert r[0] == ref[0] and r[1] == ref[1], m
        for a, b in zip(r[2:], ref[2:]):
            for k in GROUPS:
                assert np.array_equal(a[k], b[k]), (m, k)
    # several views per iteration (the all-views variant: gradients summed, k_chain + k_adam)
    plan2 = [[[0, 1], [1, 2], [2, 0]], [[1, 2], [0, 1], [0, 2]]]
    r2 = {m: _run_round(G, gd, cam, views, plan2, m, s) for m in ("steps", "graph")}
    assert r2["graph"][0] == r2["steps"][0] == 6 and r2["graph"][1] == r2["steps"][1]
    for a, b in zip(r2["graph"][2:], r2["steps"][2:]):
        for k in GROUPS:
            assert np.array_equal(a[k], b[k]), ("multi-view", k)
    # the parameters did move (the window sees Gaussians)
    g0 = G.Gaussians.from_dict(gd).to_numpy()
    assert any(not np.array_equal(ref[2][k], g0[k]) for k in GROUPS)


def test_refine_round_full_size_graph_matches_direct():
    """The same at cfg4 size (3600 tiles; gradients arrive by fp32 atomics from many tiles, so
    the two schedules agree to rounding): losses within 1e-5 relative, parameters within
    2 lr per iteration."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg4")
    frs = H.frames(cfg, 2, start=30)
    cam, views = _round_views(G, cfg, frs, (0, 0, cfg.width, cfg.height))
    gd = S.make_gaussians(cfg, n=40000, sh_degree=3)
    plan = [[[i % 2] for i in range(4)]] * 2
    s = torch.cuda.Stream()
    a = _run_round(G, gd, cam, views, plan, "graph", s)
    b = _run_round(G, gd, cam, views, plan, "direct", s)
    assert a[0] == b[0] == 8
    assert np.allclose(a[1], b[1], rtol=1e-5, atol=0)
    lr = {"xyz": 1.6e-4, "log_scale": 5e-3, "rot": 1e-3, "opacity_raw": 5e-2, "sh": 2.5e-3}
    for k in GROUPS:
        assert np.max(np.abs(np.asarray(a[2][k], np.float64) - b[2][k])) <= 2 * 8 * lr[k], k


def test_refine_round_rejects_bad_view_index_and_keeps_state():
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2")
    frs = H.frames(cfg, 1, start=4)
    cam, views = _round_views(G, cfg, frs, (312, 232, 16, 16))
    g = G.Gaussians.from_dict(S.make_gaussians(cfg, n=500))
    st = G.AdamState(g)
    ras = G.Rasterizer(g.n, cam, G.RenderConfig())
    s = torch.cuda.Stream()
    for graph in (True, False):
        with pytest.raises(G._native.GPSError):
            ras.refine_round(g, st, views, [[0], [1]], graph=graph, stream=s)
        assert st.step == 0
    ras.refine_round(g, st, views, [], graph=True, stream=s)  # an empty round is a no-op
    assert st.step == 0


def test_refine_round_graph_as_the_first_call_of_a_process():
    """The library's once-per-process setup (the host-mapped overflow flag, kernel attributes)
    happens before the capture even when a graph round is the process's first render call."""
    import os
    import subprocess
    import sys
    code = (
        "import torch, numpy as np, gps_synth as S, paper_2509_11574_b200 as G\n"
        "from tests.test_gpu_render_refine import _round_views\n"
        "cfg = S.get_config('cfg2'); frs = S.make_frames(cfg, 2, start=4, device='cpu')\n"
        "cam, views = _round_views(G, cfg, frs, (0, 0, cfg.width, cfg.height))\n"
        "g = G.Gaussians.from_dict(S.make_gaussians(cfg, n=5000)); st = G.AdamState(g)\n"
        "ras = G.Rasterizer(g.n, cam, G.RenderConfig()); s = torch.cuda.Stream()\n"
        "for r in range(3):\n"
        "    ras.refine_round(g, st, views, [[0], [1], [0]], graph=True, stream=s)\n"
        "torch.cuda.synchronize(); assert st.step == 9 and ras.loss.item() > 0\n"
        "print('OK')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stderr[-2000:]


def test_refine_round_graph_error_inside_capture_leaves_stream_usable():
    """A workspace too small for the round is found inside the capture: the capture ends, nothing
    is launched, the step count is unchanged, and the next round on the same stream runs."""
    import paper_2509_11574_b200 as G
    cfg = S.get_config("cfg2")
    frs = H.frames(cfg, 2, start=4)
    cam, views = _round_views(G, cfg, frs, (0, 0, cfg.width, cfg.height))
    g = G.Gaussians.from_dict(S.make_gaussians(cfg, n=4000))
    st = G.AdamState(g)
    ras = G.Rasterizer(g.n, cam, G.RenderConfig())
    good = ras.ws
    ras.ws = good[: good.numel() // 4]  # too small
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with pytest.raises(G._native.GPSError):
        ras.refine_round(g, st, views, [[0], [1]], graph=True, stream=s)
    assert st.step == 0
    ras.ws = good
    ras.refine_round(g, st, views, [[0], [1]], graph=True, stream=s)
    torch.cuda.synchronize()
    assert st.step == 2 and ras.loss.item() > 0
