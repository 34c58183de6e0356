#!/usr/bin/env python3
"""Per-ray march statistics of gps_raycast on a steady-state cfg4 volume (diagnostics only:
GPS_RAYCAST_DEBUG=1 makes the vertex output carry iterations / block skips / invalid samples)."""
import os
import sys

os.environ["GPS_RAYCAST_DEBUG"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gps_synth as S  # noqa: E402
import paper_2509_11574_b200 as G  # noqa: E402

cfg = S.get_config("cfg4")
scene = S.make_scene(cfg)
dc = S.pixel_rays(cfg, "cuda")
poses = S.trajectory(cfg, 62)
vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots)
cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
for k in range(60):
    f = S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc)
    vol.fuse(cam, f.R, f.t, f.depth, cfg.depth_scale, f.rgba)
f = S.render_frame(cfg, scene, *poses[60], k=60, device="cuda", dc=dc)
D, C, V = vol.raycast(cam, f.R, f.t, want_vertex=True)
torch.cuda.synchronize()
V = V.cpu().numpy()
it, sk, inv = V[..., 0], V[..., 1], V[..., 2]
D = D.cpu().numpy()
print("iterations: mean %.1f p50 %d p90 %d p99 %d max %d" % (it.mean(), *np.percentile(it, [50, 90, 99, 100])))
print("skips: mean %.1f p90 %d max %d ; invalid samples: mean %.1f p90 %d max %d" % (
    sk.mean(), np.percentile(sk, 90), sk.max(), inv.mean(), np.percentile(inv, 90), inv.max()))
# warp-level cost: each warp = 16x2 pixels; cost = max over its lanes
Wt = it.reshape(cfg.height // 2, 2, cfg.width // 16, 16).max(axis=(1, 3))
print("warp max iterations: mean %.1f; lane efficiency %.3f" % (Wt.mean(), it.mean() / Wt.mean()))
long = it > np.percentile(it, 99)
ys, xs = np.nonzero(long)
print("long rays: n", long.sum(), "hit frac", (D[long] > 0).mean(), "depth mean", D[long][D[long] > 0].mean(),
      "skips", sk[long].mean(), "invalid", inv[long].mean())
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "raystats.npz"), it=it, sk=sk, inv=inv, D=D,
                    gt=f.depth_m.cpu().numpy())
