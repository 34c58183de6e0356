"""Diagnostic: worst per-component gradient errors of the refine step against the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import gps_synth as S
import oracle as O
import paper_2509_11574_b200 as G
from tests.test_gpu_render_refine import oracle_grads, setup, GROUPS


def report(gg, ref, gamb, gd):
    keep = ~gamb
    for k in GROUPS:
        a = gg[k].reshape(len(keep), -1)
        b = ref[k].reshape(len(keep), -1)
        tau = 1e-3 * np.max(np.abs(b[keep]))
        err = np.abs(a - b) / np.maximum(np.abs(b), tau)
        err[~keep] = 0
        i, j = np.unravel_index(np.argmax(err), err.shape)
        vec = np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), tau)
        vec[~keep] = 0
        print(f"{k:12s} max comp err {err.max():.3e} at g{i}[{j}] gpu {a[i]} ref {b[i]} | vec err max {vec.max():.3e} "
              f"| group max {np.abs(b[keep]).max():.3e}")
        if k == "rot":
            q = gd["rot"][i]; s = np.exp(gd["log_scale"][i])
            print("   q", q, "|q|", np.linalg.norm(q), "scales", s, "op", gd["opacity_raw"][i])
            order = np.argsort(-err.max(1))[:8]
            for o in order:
                print("   ", o, f"{err[o].max():.2e}", "scales", np.exp(gd['log_scale'][o]), "|b|", np.abs(b[o]).max(), "|dls|", np.abs(ref['log_scale'].reshape(len(keep),-1)[o]).max())


def run(gd, c, gcam, R, t, Dt, Ct, tgt):
    dev = dict(Dt=torch.from_numpy(Dt).cuda(), Ct=torch.from_numpy(Ct).cuda(), tgt=torch.from_numpy(np.asarray(tgt)).cuda())
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig(tile_depth_precull=0))
    ras.refine_step(g, st, [G.View(gcam, R, t, dev["Dt"], dev["Ct"], dev["tgt"])], grad_out=gout)
    oloss, ref, gamb = oracle_grads(gd, c, R, t, Dt, Ct, np.asarray(tgt))
    report(gout.to_numpy(), ref, gamb, gd)


rng = np.random.default_rng(5)
c = O.Camera(120.0, 120.0, 79.5, 59.5, 160, 120)
gcam = G.Camera(120.0, 120.0, 79.5, 59.5, 160, 120)
R, t = np.eye(3, dtype=np.float32), np.zeros(3, np.float32)
gd = S.random_gaussians(300, 1, rng, center=(0, 0, 1.0), spread=0.4, scale=(0.005, 0.12))
Dt = rng.uniform(1.1, 1.5, (120, 160)).astype(np.float32)
Ct = rng.random((120, 160, 3)).astype(np.float32)
tgt = rng.integers(0, 256, (120, 160, 4)).astype(np.uint8)
print("== large"); run(gd, c, gcam, R, t, Dt, Ct, tgt)
Gm, cfg, fr, gd, Dt, Ct, tgt, gcam, ocam, dev = setup()
nc = 4
gd = dict(gd, sh_degree=1, sh=np.ascontiguousarray(gd["sh"].reshape(len(gd["xyz"]), 16, 3)[:, :nc].reshape(-1, 3 * nc)))
print("== sh1"); run(gd, ocam, gcam, fr.R, fr.t, Dt, Ct, tgt)
