"""Edge cases of the GPU path against the CPU oracle (③: ragged inputs, maximum sizes, degenerate
cases).

* A ragged 100x75 image (tiles and warps straddle the right and bottom borders, the pixel count
  is no multiple of any block size) through fuse, raycast, render and the refine gradients.
* A tile list longer than both shared-memory sorts (> 2048 entries in one tile): the global
  bitonic fallback keeps the lists bit-exact and the image and gradients equal to the oracle's.
* An SDF render that missed everywhere (D_t = 0: no depth test, C_t = 0, R-MISS).
Bars as in test_gpu_fuse_raycast.py / test_gpu_render_refine.py."""
import numpy as np
import pytest
import torch

import gps_synth as S
import oracle as O
from tests import gpu_helpers as H
from tests.test_gpu_fuse_raycast import compare_volumes, raycast_compare
from tests.test_gpu_render_refine import check_forward, compare_grads, oracle_grads

pytestmark = pytest.mark.gpu


def _ragged_cfg():
    # cfg2's room and noise at a ragged 100x75, intrinsics scaled from cfg2's field of view
    return S.get_config("cfg2", width=100, height=75, fx=82.0, fy=82.0, cx=49.5, cy=37.0)


def test_ragged_image_fuse_and_raycast():
    cfg = _ragged_cfg()
    frs = H.frames(cfg, 2)
    gvol, ovol = H.fuse_both(cfg, frs)
    compare_volumes(gvol, ovol, 20)
    raycast_compare(cfg, gvol, ovol, frs[1].R, frs[1].t)


@pytest.mark.parametrize("sort_free", [0, 1])
def test_ragged_image_render_and_gradients(sort_free):
    import paper_2509_11574_b200 as G
    cfg = _ragged_cfg()
    fr = H.frames(cfg, 1)[0]
    gd = S.make_gaussians(cfg, n=3000, frames=[fr])
    Dt, Ct = S.sdf_stage_inputs(cfg, fr)
    tgt = fr.rgba
    gcam, ocam = H.cams(cfg)
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=tgt.cuda().contiguous())
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(sort_free=sort_free))
    Cs, W, loss = ras.render(g, gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    out = O.render(gd, ocam, fr.R, fr.t, Dt, Ct)
    check_forward(out, Cs.cpu().numpy(), W.cpu().numpy())
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras.refine_step(g, st, [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, ocam, fr.R, fr.t, Dt, Ct, tgt.numpy())
    compare_grads(gout.to_numpy(), ref, gamb, min_checked=100)


def _crowded(n=2600):
    """n Gaussians crowding one 16x16 tile of a 96x64 view: that tile's list exceeds both
    shared-memory sorts (256 for the rank sort, 2048 for the one-pixel kernel's bitonic)."""
    rng = np.random.default_rng(11)
    c = O.Camera(80.0, 80.0, 47.5, 31.5, 96, 64)
    gd = S.random_gaussians(n, 1, rng, center=(0.0, 0.0, 1.0), spread=0.004, scale=(0.002, 0.006))
    gd["opacity_raw"] = np.full(n, -2.0, np.float32)  # sigma ~ 0.12: many small contributions
    return c, gd, rng


def test_tile_list_beyond_shared_memory_sorts():
    import paper_2509_11574_b200 as G
    c, gd, rng = _crowded()
    gcam = G.Camera(80.0, 80.0, 47.5, 31.5, 96, 64)
    R, t = np.eye(3, dtype=np.float32), np.zeros(3, np.float32)
    Dt = np.zeros((64, 96), np.float32)  # no SDF surface: every entry is in front (R-MISS)
    Ct = rng.random((64, 96, 3)).astype(np.float32)
    Ct[:] = 0.0
    tgt = rng.integers(0, 256, (64, 96, 4)).astype(np.uint8)
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=torch.from_numpy(tgt).cuda())
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile_depth_precull=0))
    Cs, W, loss = ras.render(g, gcam, R, t, dev["Dt"], dev["Ct"], dev["tgt"])
    gv, grng = ras.lists()
    lens = grng[:, 1] - grng[:, 0]
    assert lens.max() > 2048
    rect, depth, culled = O.project_p32(gd, c, R, t, O.RenderCfg())
    ov, orng = O.tile_lists(rect, depth, culled, 96, 64, 16)
    assert np.array_equal(grng, orng) and np.array_equal(gv, ov)
    out = O.render(gd, c, R, t, Dt, Ct)
    check_forward(out, Cs.cpu().numpy(), W.cpu().numpy())
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras.refine_step(g, st, [G.View(gcam, R, t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, c, R, t, Dt, Ct, tgt)
    compare_grads(gout.to_numpy(), ref, gamb, min_checked=500)


def test_pair_capacity_overflow_is_reported_and_contained():
    """max_pairs below the frame's (tile, entry) count: the render reports
    GPS_ERR_WORKSPACE_TOO_SMALL through gps_render_stats_sync, writes nothing past the pair
    capacity (a guard region after the workspace stays intact), and a render with enough
    capacity on the same Gaussians still matches the oracle."""
    import paper_2509_11574_b200 as G
    cfg = _ragged_cfg()
    fr = H.frames(cfg, 1)[0]
    gd = S.make_gaussians(cfg, n=3000, frames=[fr])
    Dt, Ct = S.sdf_stage_inputs(cfg, fr)
    gcam, ocam = H.cams(cfg)
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=fr.rgba.cuda().contiguous())
    g = G.Gaussians.from_dict(gd)
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(max_pairs=64))
    n_ws = ras.ws.numel()
    guard = torch.full((1 << 16,), 0xA5, dtype=torch.uint8, device="cuda")
    big = torch.cat([ras.ws, guard])  # the workspace followed by a guard region
    ras.ws = big[:n_ws]
    ras.render(g, gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    st = ras.stats()
    assert st["status"] == "GPS_ERR_WORKSPACE_TOO_SMALL" and st["pairs"] > st["capacity"] == 64
    assert bool((big[n_ws:] == 0xA5).all())
    ok = G.Rasterizer(g.n, gcam, G.RenderConfig())
    Cs, W, _ = ok.render(g, gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    assert ok.stats()["status"] == "GPS_OK"
    check_forward(O.render(gd, ocam, fr.R, fr.t, Dt, Ct), Cs.cpu().numpy(), W.cpu().numpy())


def test_pair_overflow_in_an_earlier_view_is_sticky():
    """an overflow in the FIRST view of a multi-view refine step is not lost when a
    later view fits: the host-mapped sticky flag makes the next render / refine call return
    GPS_ERR_WORKSPACE_TOO_SMALL (once), after which calls succeed again."""
    import paper_2509_11574_b200 as G
    cfg = _ragged_cfg()
    fr = H.frames(cfg, 1)[0]
    gd = S.make_gaussians(cfg, n=3000, frames=[fr])
    Dt, Ct = S.sdf_stage_inputs(cfg, fr)
    gcam, _ = H.cams(cfg)
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=fr.rgba.cuda().contiguous())
    g = G.Gaussians.from_dict(gd)
    # view 1 sees the Gaussians (overflows 64 pairs), view 2 looks away (0 pairs)
    Rb = np.array([[-1, 0, 0], [0, 1, 0], [0, 0, -1]], np.float32) @ np.asarray(fr.R, np.float32)
    views = [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"]),
             G.View(gcam, Rb, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])]
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(max_pairs=64), n_views=2)
    st = G.AdamState(g)
    ras.refine_step(g, st, views)
    torch.cuda.synchronize()
    with pytest.raises(G._native.GPSError) as e:
        ras.refine_step(g, st, views[1:])
    assert e.value.status == 3
    ras.refine_step(g, st, views[1:])  # reported once: the next call runs
    torch.cuda.synchronize()


def test_tracking_rejects_bad_configs():
    import paper_2509_11574_b200 as G
    from paper_2509_11574_b200 import _native as N
    cfg = _ragged_cfg()
    fr = H.frames(cfg, 1)[0]
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    V = torch.zeros((cfg.height, cfg.width, 3), dtype=torch.float32, device="cuda")
    eye = np.eye(3, dtype=np.float32)
    for bad in (dict(levels=0), dict(levels=5), dict(filter_radius=9), dict(min_pivot_ratio=-1.0),
                dict(filter_radius=2, filter_sigma_r=0.0)):
        with pytest.raises(N.GPSError):
            G.track(cam, fr.depth.cuda(), cfg.depth_scale, V, V, eye, np.zeros(3), eye, np.zeros(3),
                    G.IcpConfig(**bad))


def test_empty_gaussian_set():
    """N = 0 (no preprocess launch): the render is the SDF image itself (C* = C_t, W_G = 0, no
    pairs), the loss is the oracle's, and a refine step is a no-op that still counts the step."""
    import paper_2509_11574_b200 as G
    cfg = _ragged_cfg()
    fr = H.frames(cfg, 1)[0]
    gd = S.make_gaussians(cfg, n=0, frames=[fr])
    Dt, Ct = S.sdf_stage_inputs(cfg, fr)
    gcam, ocam = H.cams(cfg)
    tgt = fr.rgba.numpy()
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=fr.rgba.cuda().contiguous())
    g = G.Gaussians.from_dict(gd)
    assert g.n == 0
    ras = G.Rasterizer(max(g.n, 1), gcam, G.RenderConfig())
    Cs, W, loss = ras.render(g, gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])
    assert np.array_equal(Cs.cpu().numpy(), Ct) and not W.cpu().numpy().any()
    assert ras.stats()["pairs"] == 0
    out = O.render(gd, ocam, fr.R, fr.t, Dt, Ct)
    ol, _, _, _ = O.l1_loss(out["Cstar"], out["WG"], Dt, tgt)
    assert abs(loss.item() - ol) <= 1e-5 * max(ol, 1e-6)
    st = G.AdamState(g)
    ras.refine_step(g, st, [G.View(gcam, fr.R, fr.t, dev["Dt"], dev["Ct"], dev["tgt"])])
    assert st.step == 1
