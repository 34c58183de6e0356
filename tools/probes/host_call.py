# host cost of one gps_refine_step call: the Python wrapper vs the bare ctypes call with prebuilt
# arguments (no synchronisation inside the timed loops)
import ctypes as C, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import gps_synth as S, paper_2509_11574_b200 as G
from paper_2509_11574_b200 import api as A, _native as N
cfg = S.get_config("cfg2")
fr = S.make_frames(cfg, 1, start=5)[0]
gd = S.make_gaussians(cfg, n=20000)
Dt, Ct = S.sdf_stage_inputs(cfg, fr, seed=5)
cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
g = G.Gaussians.from_dict(gd); st = G.AdamState(g)
ras = G.Rasterizer(g.n, cam, G.RenderConfig())
view = G.View(cam, fr.R, fr.t, torch.from_numpy(Dt).cuda(), torch.from_numpy(Ct).cuda(), fr.rgba.cuda().contiguous())
for _ in range(5): ras.refine_step(g, st, [view])
torch.cuda.synchronize()
n = 100
t0 = time.perf_counter()
for _ in range(n): ras.refine_step(g, st, [view])
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
arr = (N.gps_view * 1)(view.c()); sa = N.gps_adam_state(st.m.c(), st.v.c(), st.step); gc = g.c()
rc = ras.cfg.c(); ac = G.AdamConfig().c(); s = torch.cuda.current_stream().cuda_stream
wsp = A._ptr(ras.ws); lp = A._ptr(ras.loss)
t3 = time.perf_counter()
for _ in range(n):
    A._L.gps_refine_step(C.byref(gc), C.byref(sa), arr, 1, C.byref(rc), C.byref(ac), wsp, ras.ws.numel(), lp, None, s)
t4 = time.perf_counter()
torch.cuda.synchronize()
t5 = time.perf_counter()
print(f"wrapper {1e6*(t1-t0)/n:.1f} us/call (device {1e6*(t2-t0)/n:.1f}); bare ctypes {1e6*(t4-t3)/n:.1f} us/call (device {1e6*(t5-t3)/n:.1f})")
