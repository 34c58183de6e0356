"""Chained end-to-end parity: the CUDA path and the CPU oracle each start from the
same raw frames and run the whole mapping step on their OWN intermediate results --
fuse -> raycast (D_t, C_t at the view pose) -> render (Eqs. 1-4 over C_t) -> L1 -> backward ->
Adam -- compared stage by stage.  Nothing either side computes feeds the other.

Ambiguity rule: a pixel is excluded (and counted) when its raycast is an
fp32 near-tie or differs between the sides (at most 1e-4 of the pixels may differ outside
near-ties), or when a Gaussian's depth test d < D_t + eps at that pixel is closer to its threshold
than the two sides' D_t differ there (both outcomes are correct).  Gaussians with an in-pair at
an excluded pixel are excluded from the gradient comparison.  PAPER.md P:70-73, P:75-97, P:106,
P:140."""
import numpy as np
import pytest
import torch

import gps_synth as S
import oracle as O
from tests import gpu_helpers as H
from tests.test_gpu_fuse_raycast import TIE_VOXELS, compare_volumes
from tests.test_gpu_render_refine import GROUPS, compare_grads, grad_sensitivity

pytestmark = pytest.mark.gpu

EPS = 0.02


def depth_test_ties(gd, ocam, R, t, Dg, Do, excl):
    """pixels where some non-culled Gaussian's rect covers the pixel and |d - (D_o + eps)| is
    within the two sides' depth difference (+1e-6 m): its membership may differ legitimately."""
    rect, d, culled = O.project_p32(gd, ocam, R, t, O.RenderCfg())
    tol = np.abs(Dg - Do) + 1e-6
    thr = np.where(Do > 0, Do + EPS, np.inf)
    out = excl.copy()
    for i in np.nonzero(culled == 0)[0]:
        x0, y0, x1, y1 = rect[i]
        if x1 < x0 or y1 < y0:
            continue
        sl = (slice(y0, y1 + 1), slice(x0, x1 + 1))
        out[sl] |= np.abs(float(d[i]) - thr[sl]) <= tol[sl]
    return out


def report_grads(label, gg, ref, gamb):
    keep = ~gamb
    msg = []
    for k in GROUPS:
        a = gg[k].reshape(len(keep), -1)[keep]
        b = ref[k].reshape(len(keep), -1)[keep]
        tau = 1e-3 * np.max(np.abs(b))
        err = np.abs(a - b) / np.maximum(np.abs(b), tau)
        i = np.unravel_index(np.argmax(err), err.shape)
        gi = np.nonzero(keep)[0][i[0]]
        msg.append(f"{k}: max {err.max():.2e} (Gaussian {gi}, gpu {a[i]:.4e} ref {b[i]:.4e} tau {tau:.3e})")
    print(f"grads {label}: {int(keep.sum())} compared; " + "; ".join(msg))


def run_chain(cfg_name, n_frames, n_gauss=None):
    import paper_2509_11574_b200 as G
    cfg = S.get_config(cfg_name)
    frs = H.frames(cfg, n_frames)
    gcam, ocam = H.cams(cfg)
    # (a2, a3) fuse on both sides from the same raw frames
    gvol, ovol = H.fuse_both(cfg, frs)
    compare_volumes(gvol, ovol, 50)
    view = frs[-1]
    R, t = view.R, view.t
    # (a4) each side raycasts its own volume at the view pose
    Dg_t, Cg_t, _ = gvol.raycast(gcam, R, t)
    torch.cuda.synchronize()
    Dg = Dg_t.cpu().numpy().reshape(cfg.height, cfg.width).astype(np.float64)
    Do, Co, _, margin = ovol.raycast(ocam, R, t)
    Do = Do.reshape(cfg.height, cfg.width)
    Co = Co.reshape(cfg.height, cfg.width, 3)
    margin = margin.reshape(cfg.height, cfg.width)
    n = Dg.size
    ray_diff = ((Dg > 0) != (Do > 0)) | ((Dg > 0) & (Do > 0) & (np.abs(Dg - Do) > 1e-4))
    tie = margin < TIE_VOXELS
    assert (ray_diff & ~tie).sum() <= int(1e-4 * n)
    assert (ray_diff & tie).sum() <= max(2, int(1e-3 * n))
    excl = ray_diff.copy()  # only pixels whose raycasts actually differ
    # (a5-a9) each side renders over its OWN D_t, C_t
    gd = S.make_gaussians(cfg, n=n_gauss, frames=frs if cfg_name == "cfg1" else None)
    tgt = S.target_rgba(cfg, view)
    excl = depth_test_ties(gd, ocam, R, t, Dg, Do, excl)
    g = G.Gaussians.from_dict(gd)
    p0 = g.to_numpy()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
    Cs_g, W_g, loss_g = ras.render(g, gcam, R, t, Dg_t, Cg_t, tgt.cuda())
    out = O.render(gd, ocam, R, t, Do, Co)
    Cs_g = Cs_g.cpu().numpy().reshape(cfg.height, cfg.width, 3)
    W_g = W_g.cpu().numpy().reshape(cfg.height, cfg.width)
    keep = ~excl
    print(f"chain {cfg_name}: {n} px, {int(ray_diff.sum())} raycast differences "
          f"({int((ray_diff & tie).sum())} at near-ties), {int(excl.sum())} px excluded, "
          f"{int((out['WG'] > 0).sum())} px with W_G > 0")
    assert excl.sum() <= 0.01 * n
    assert np.max(np.abs(Cs_g[keep] - out["Cstar"][keep])) <= 1e-3
    assert np.all(np.abs(W_g[keep] - out["WG"][keep]) <= 1e-3 * out["WG"][keep] + 1e-6)
    assert out["WG"].max() > 0.5
    # (a9) L1 over each side's own mask: excluded pixels can move the mean by <= 1/|M| each
    ol, OG, cnt, samb = O.l1_loss(out["Cstar"], out["WG"], Do, tgt.numpy())
    lg = loss_g.item()
    assert abs(lg - ol) <= 1e-5 * ol + excl.sum() / cnt
    # (a10, a11) one refine iteration on each side's own view: gradients and the Adam update
    st = G.AdamState(g)
    gout = g.zeros_like()
    gview = G.View(gcam, R, t, Dg_t, Cg_t, tgt.cuda())
    l2 = ras.refine_step(g, st, [gview], grad_out=gout).item()
    assert abs(l2 - lg) <= 1e-6 * lg
    ref, gamb = O.backward(gd, ocam, R, t, Do, out["Cstar"], out["WG"], OG, pix_amb=(samb | excl))
    gg = gout.to_numpy()
    report_grads("chained", gg, ref, gamb)
    sens = grad_sensitivity(gd, ocam, R, t, Do, out["Cstar"], out["WG"], OG, samb | excl)
    compare_grads(gg, ref, gamb, sens=sens)
    m0 = {k: np.zeros_like(np.asarray(p0[k], np.float64)) for k in GROUPS}
    P1, _, _ = O.adam_step(p0, m0, m0, ref, 0)
    p1 = g.to_numpy()
    for k in GROUPS:
        b = ref[k].reshape(len(gamb), -1)
        sel = (np.abs(b) > 1e-2 * np.max(np.abs(b))) & ~gamb[:, None]
        assert sel.sum() > 0
        a1 = p1[k].reshape(len(gamb), -1)[sel]
        e1 = P1[k].reshape(len(gamb), -1)[sel]
        assert np.max(np.abs(a1 - e1)) <= 1e-6 * np.max(np.abs(e1)) + 1e-7, k
    return excl.sum(), gamb.sum()


def test_chain_cfg1():
    run_chain("cfg1", 1)


def test_chain_cfg2_three_frame_prefix():
    run_chain("cfg2", 3, n_gauss=20000)
