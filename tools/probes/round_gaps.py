# A refinement round alone (no fusion beside it) on the steady cfg4 state: graph vs direct
# launches vs the sum of its kernels' event-profiled times (the launch gaps of the round)
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import gps_synth as S, paper_2509_11574_b200 as G
from paper_2509_11574_b200 import _native as N
import bench
cfg = S.get_config("cfg4"); scene = S.make_scene(cfg); dc = S.pixel_rays(cfg, "cuda")
poses = S.trajectory(cfg, 70)
frames = [S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc) for k in range(70)]
cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots)
for k in range(60):
    f = frames[k]; vol.fuse(cam, f.R, f.t, f.depth, cfg.depth_scale, f.rgba)
g = G.Gaussians.from_dict(S.make_gaussians(cfg)); st = G.AdamState(g)
ras = G.Rasterizer(g.n, cam, G.RenderConfig())
views = []
for j, k in enumerate((20, 32, 44, 52, 56, 59)):
    D = torch.empty((cfg.height, cfg.width), device="cuda"); Cc = torch.empty((cfg.height, cfg.width, 3), device="cuda")
    vol.raycast(cam, frames[k].R, frames[k].t, D, Cc)
    views.append(G.View(cam, frames[k].R, frames[k].t, D, Cc, frames[k].rgba))
order = [[i % 6] for i in range(20)]
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
torch.cuda.synchronize()
def timed(graph):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); ras.refine_round(g, st, views, order, graph=graph, stream=s); e1.record(s)
    torch.cuda.synchronize(); return e0.elapsed_time(e1)
for rep in range(3):
    tg = [timed(True) for _ in range(3)]
    td = [timed(False) for _ in range(3)]
    print("graph", [round(x, 3) for x in tg], "direct", [round(x, 3) for x in td])
N._lib.gps_profile_enable(1)
timed(False)
prof = bench.read_profile(N)
N._lib.gps_profile_enable(0)
tot = sum(v["ms"] for v in prof.values())
print("kernel sum", round(tot, 3), {k: round(v["ms"], 3) for k, v in prof.items() if v["ms"] > 0})
