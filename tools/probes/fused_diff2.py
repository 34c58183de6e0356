import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import gps_synth as S, paper_2509_11574_b200 as G
from tests import gpu_helpers as H
GROUPS = ("xyz", "log_scale", "rot", "opacity_raw", "sh")
cfg = S.get_config("cfg2"); fr = H.frames(cfg, 1, start=5)[0]
n = 50001
gd = S.make_gaussians(cfg, n=n, sh_degree=3)
Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=5)
tgt = S.target_rgba(cfg, fr).cuda().contiguous(); gcam, _ = H.cams(cfg)
view = G.View(gcam, fr.R, fr.t, torch.from_numpy(Dt).cuda(), torch.from_numpy(Ct).cuda(), tgt)
res = {}
for mode in ("fused", "unfused"):
    if mode == "unfused": os.environ["GPS_UNFUSED_ADAM"] = "1"
    g = G.Gaussians.from_dict(gd); st = G.AdamState(g); gout = g.zeros_like()
    ras = G.Rasterizer(g.n, gcam, G.RenderConfig())
    l = ras.refine_step(g, st, [view], grad_out=gout).item(); torch.cuda.synchronize()
    res[mode] = (l, g.to_numpy(), st.m.to_numpy(), st.v.to_numpy(), gout.to_numpy())
fl, fu = res["fused"], res["unfused"]
print("loss", fl[0], fu[0])
for name, i in (("p", 1), ("m", 2), ("v", 3), ("g", 4)):
    for k in GROUPS:
        a, b = np.asarray(fl[i][k], np.float64).reshape(n, -1), np.asarray(fu[i][k], np.float64).reshape(n, -1)
        bad = ~(np.abs(a - b) <= 1e-4 * np.abs(b) + 1e-6 * np.abs(b).max())
        nzd = (a != 0) != (b != 0)
        if bad.any() or nzd.any():
            r, c = np.nonzero(bad | nzd)
            print(name, k, bad.sum(), nzd.sum(), "rows", r[:8], "cols", c[:8], a[r[0], c[0]], b[r[0], c[0]])
