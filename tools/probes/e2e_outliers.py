# host time per call on the end-to-end path (pinned host frames), cfg4, several windows: where do
# the host stalls of a collapsed end-to-end window go?
import os, sys, time, collections
sys.path.insert(0, os.getcwd())
import torch
import gps_synth as S, paper_2509_11574_b200 as G
from paper_2509_11574_b200.pipeline import MappingPipeline
torch.cuda.set_stream(torch.cuda.Stream())
T = collections.defaultdict(list)
def wrap(obj, name, key):
    f = getattr(obj, name)
    def w(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[key].append(time.perf_counter() - t0); return r
    setattr(obj, name, w)
cfg = S.get_config("cfg4"); scene = S.make_scene(cfg); dc = S.pixel_rays(cfg, "cuda")
n = 60 + 10 * 45
poses = S.trajectory(cfg, n)
frames = [S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc) for k in range(n)]
cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots)
g = G.Gaussians.from_dict(S.make_gaussians(cfg))
ahead = int(os.environ.get("AHEAD", "20"))
pipe = MappingPipeline(cam, g, vol, cfg.depth_scale, max_frames_ahead=ahead)
if os.environ.get("PREWARM"):
    with torch.cuda.stream(pipe.copy_stream):
        tmp = torch.empty(int(os.environ["PREWARM"]) << 20, dtype=torch.uint8, device="cuda")
    del tmp
for k in range(60):
    f = frames[k]; pipe.process_frame(k, f.depth, f.rgba, f.R, f.t, refine=False)
host = {k: (frames[k].depth.cpu().pin_memory(), frames[k].rgba.cpu().pin_memory()) for k in range(60, n)}
import ctypes
for obj, name, key in ((pipe, "_upload", "upload"), (pipe.vol, "fuse_raycast", "fuse_raycast"),
                       (pipe.vol, "raycast", "raycast"), (pipe.ras, "refine_round", "refine_round"),
                       (pipe.kf, "offer", "kf.offer"), (pipe, "_drop_frames", "drop")):
    wrap(obj, name, key)
PF = []
def run(k0, k1):
    for k in range(k0, k1):
        f = frames[k]
        t0 = time.perf_counter()
        pipe.process_frame(k, host[k][0], host[k][1], f.R, f.t, prefetch=host.get(k + 1))
        PF.append(time.perf_counter() - t0)
run(60, 110); pipe.join(); torch.cuda.synchronize()
for w in range(4):
    T.clear(); PF.clear(); w0 = pipe.host_wait_s; a0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    k0 = 110 + 100 * w
    t0 = time.perf_counter(); run(k0, k0 + 100); t1 = time.perf_counter(); pipe.join(); torch.cuda.synchronize(); t2 = time.perf_counter()
    wait = pipe.host_wait_s - w0
    print(f"window {w}: host {100*(t1-t0):.2f} ms/step (wait {100*wait:.2f}), wall {100*(t2-t0):.2f} ms/step; "
          f"process_frame max {1000*max(PF):.2f} ms, p50 {1000*sorted(PF)[50]:.3f}, "
          f"cudaMallocs {torch.cuda.memory_stats().get('num_device_alloc', 0) - a0}")
    for key, v in sorted(T.items(), key=lambda x: -sum(x[1])):
        v = sorted(v)
        print(f"   {key:13s} n={len(v):4d} sum {1000*sum(v)/10:.3f} ms/step  p50 {1e6*v[len(v)//2]:.0f} us  max {1e6*v[-1]:.0f} us")
