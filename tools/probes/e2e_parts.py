# host time per part of process_frame on the end-to-end path (pinned host frames), cfg4
import os, sys, time, collections
sys.path.insert(0, os.getcwd())
import torch
import gps_synth as S, paper_2509_11574_b200 as G
from paper_2509_11574_b200 import pipeline as PL
from paper_2509_11574_b200.pipeline import MappingPipeline
T = collections.defaultdict(float)
def wrap(obj, name, key):
    f = getattr(obj, name)
    def w(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[key] += time.perf_counter() - t0; return r
    setattr(obj, name, w)
cfg = S.get_config("cfg4"); scene = S.make_scene(cfg); dc = S.pixel_rays(cfg, "cuda")
n = 60 + 10 * 12
poses = S.trajectory(cfg, n)
frames = [S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc) for k in range(n)]
cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots)
g = G.Gaussians.from_dict(S.make_gaussians(cfg))
pipe = MappingPipeline(cam, g, vol, cfg.depth_scale)
for k in range(60):
    f = frames[k]; pipe.process_frame(k, f.depth, f.rgba, f.R, f.t, refine=False)
host = {k: (frames[k].depth.cpu().pin_memory(), frames[k].rgba.cpu().pin_memory()) for k in range(60, n)}
for obj, name, key in ((pipe, "_upload", "upload"), (pipe, "_device", "device"), (pipe.vol, "fuse", "fuse"),
                       (pipe.vol, "raycast", "raycast"), (pipe.ras, "refine_step", "refine_step"),
                       (pipe.kf, "offer", "kf.offer"), (pipe, "_refine_round", "round(total)")):
    wrap(obj, name, key)
def run(k0, k1):
    for k in range(k0, k1):
        f = frames[k]
        pipe.process_frame(k, host[k][0], host[k][1], f.R, f.t, prefetch=host.get(k + 1))
run(60, 100); pipe.join(); torch.cuda.synchronize()
T.clear()
t0 = time.perf_counter(); run(100, 160); t1 = time.perf_counter(); pipe.join(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host {1000*(t1-t0)/6:.2f} ms/step, wall {1000*(t2-t0)/6:.2f} ms/step")
for k, v in sorted(T.items(), key=lambda x: -x[1]): print(f"  {k:14s} {1000*v/6:.3f} ms/step")
