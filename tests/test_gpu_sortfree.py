"""GPU parity of the paper's sort-free renderer (RenderConfig.sort_free = 1; PAPER.md P:99-100,
App. B, Table 7) against the same CPU oracle as the sorted
path: Eqs. 1-3 are order-free sums, so C*, W_G, the loss and the raw-parameter gradients have
the same plain definitions (O7-O9) whatever order the entries are summed in.

Bars as in test_gpu_render_refine.py: C* within 1e-3 absolute, W_G within 1e-3 relative, loss
within 1e-5 relative, gradients within 1e-3 relative with the floor 1e-3 max|g| per block.  The
tile lists hold the same (tile, Gaussian) pairs as the oracle's binning, in bucket order: they
are compared as per-tile sets, bit-exact."""
import numpy as np
import pytest
import torch

import gps_synth as S
import oracle as O
from tests import gpu_helpers as H
from tests.test_gpu_render_refine import check_forward, compare_grads, oracle_grads, setup

pytestmark = pytest.mark.gpu


def render(G, gd, gcam, fr, dev, tile=16, sort_free=1):
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile=tile, sort_free=sort_free))
    Cs, W, loss = ras.render(g, gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    torch.cuda.synchronize()
    return ras, Cs.cpu().numpy(), W.cpu().numpy(), loss.item()


@pytest.mark.parametrize("tile", [16, 8])
def test_sortfree_render_matches_oracle_and_lists_are_the_same_sets(tile):
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    ras, Cs, W, loss = render(G, gd, gcam, fr, dev, tile=tile)
    out = O.render(gd, ocam, fr.R, fr.t, Dt, Ct)
    check_forward(out, Cs, W)
    ol = O.l1_loss(out["Cstar"], out["WG"], Dt, tgt)[0]
    assert abs(loss - ol) <= 1e-5 * ol
    rect, depth, culled = O.project_p32(gd, ocam, fr.R, fr.t, O.RenderCfg())
    ov, orng = O.tile_lists(rect, depth, culled, cfg.width, cfg.height, tile)
    gv, grng = ras.lists()
    # same buckets, and no early termination: every listed entry stays in its tile's list
    assert np.array_equal(grng, orng)
    for t in range(len(orng)):
        assert np.array_equal(np.sort(gv[grng[t, 0]:grng[t, 1]]), np.sort(ov[orng[t, 0]:orng[t, 1]]))


def test_sortfree_and_sorted_images_agree():
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    _, C0, W0, l0 = render(G, gd, gcam, fr, dev, sort_free=0)
    _, C1, W1, l1 = render(G, gd, gcam, fr, dev, sort_free=1)
    assert np.max(np.abs(C1 - C0)) <= 1e-5
    assert np.all(np.abs(W1 - W0) <= 1e-5 * W0 + 1e-7)
    assert abs(l1 - l0) <= 1e-5 * l0


@pytest.mark.parametrize("tile,backward", [(16, 0), (8, 0), (16, 1), (8, 1)])
def test_sortfree_refine_gradients_match_oracle(tile, backward):
    """backward 0: the paper's thread-per-group scheme; 1: the warp-per-entry backward on the
    unsorted lists (order-free: no transmittance)."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile=tile, sort_free=1, backward=backward))
    ras.refine_step(g, st, [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt)
    compare_grads(gout.to_numpy(), ref, gamb)


def test_sortfree_large_gaussians_span_many_tiles():
    """Footprints of hundreds of pixels per tile are cut into several pixel groups, each a
    thread with its own reduction: gradients still equal the oracle's."""
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
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile_depth_precull=0, sort_free=1))
    Cs, W, loss = ras.render(g, gcam, R, t, dev["Dt"], dev["Ct"], dev["tgt"])
    out = O.render(gd, c, R, t, Dt, Ct)
    check_forward(out, Cs.cpu().numpy(), W.cpu().numpy())
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras.refine_step(g, st, [G.View(gcam, R, t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, c, R, t, Dt, Ct, tgt)
    compare_grads(gout.to_numpy(), ref, gamb, min_checked=20)


@pytest.mark.slow
def test_sortfree_full_size_cfg4():
    """The sort-free renderer at the bench's full size (1280x720, 200k Gaussians): image, loss and
    raw-parameter gradients against the oracle."""
    G, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup("cfg4", start=300)
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(sort_free=1))
    Cs, W, loss = ras.render(g, gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    out = O.render(gd, ocam, fr.R, fr.t, Dt, Ct)
    check_forward(out, Cs.cpu().numpy(), W.cpu().numpy())
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras.refine_step(g, st, [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb, sens = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt, with_sens=True)
    assert abs(loss.item() - oloss) <= 1e-5 * oloss
    compare_grads(gout.to_numpy(), ref, gamb, min_checked=10000, sens=sens)
