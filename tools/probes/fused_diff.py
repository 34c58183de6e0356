import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import gps_synth as S, paper_2509_11574_b200 as G
from tests import gpu_helpers as H
GROUPS = ("xyz", "log_scale", "rot", "opacity_raw", "sh")
cfg = S.get_config("cfg2")
fr = H.frames(cfg, 1, start=5)[0]
gd = S.make_gaussians(cfg, n=50001, sh_degree=3)
Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=5)
tgt = S.target_rgba(cfg, fr).cuda().contiguous()
gcam, _ = H.cams(cfg)
view = G.View(gcam, fr.R, fr.t, torch.from_numpy(Dt).cuda(), torch.from_numpy(Ct).cuda(), tgt)
res = {}
for mode in ("fused", "unfused"):
    if mode == "unfused": os.environ["GPS_UNFUSED_ADAM"] = "1"
    g = G.Gaussians.from_dict(gd); st = G.AdamState(g); gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
    ls = [ras.refine_step(g, st, [view], grad_out=gout).item() for _ in range(1)]
    torch.cuda.synchronize()
    res[mode] = (ls, g.to_numpy(), st.m.to_numpy(), st.v.to_numpy(), gout.to_numpy())
print(res["fused"][0], res["unfused"][0])
for name, a, b in zip(["p","m","v","g"], res["fused"][1:], res["unfused"][1:]):
    for k in GROUPS:
        x, y = np.asarray(a[k]).reshape(50001, -1), np.asarray(b[k]).reshape(50001, -1)
        d = x != y
        if d.any():
            r, c = np.nonzero(d)
            print(name, k, d.sum(), "rows", np.unique(r)[:10], "cols", np.unique(c)[:10], x[r[0], c[0]], y[r[0], c[0]])
