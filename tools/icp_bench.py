"""Times gps_track_sync on a cfg4 frame pair (model maps from the generator's analytic trace):
per-frame ICP time with CUDA events.  For ncu: `--frames 1`.

    python tools/icp_bench.py [--config cfg4] [--frames 20]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gps_synth as S  # noqa: E402
import paper_2509_11574_b200 as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--frames", type=int, default=20)
    a = ap.parse_args()
    cfg = S.get_config(a.config)
    scene = S.make_scene(cfg)
    dc = S.pixel_rays(cfg, "cuda")
    poses = S.trajectory(cfg, 2)
    f0 = S.render_frame(cfg, scene, *poses[0], k=0, device="cuda", dc=dc)
    f1 = S.render_frame(cfg, scene, *poses[1], k=1, device="cuda", dc=dc)
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots,
                   dense_bounds=S.scene_bounds(cfg))
    for _ in range(3):
        vol.fuse(cam, f0.R, f0.t, f0.depth, cfg.depth_scale, f0.rgba)
    d, c, V = vol.raycast(cam, f0.R, f0.t, want_vertex=True)
    N = G.vertex_normals(cam, f0.R, f0.t, d, V)
    res = G.track(cam, f1.depth, cfg.depth_scale, V, N, f0.R, f0.t, f0.R, f0.t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.frames):
        res = G.track(cam, f1.depth, cfg.depth_scale, V, N, f0.R, f0.t, f0.R, f0.t)
    e1.record()
    torch.cuda.synchronize()
    err = np.linalg.norm(res["t"] - np.asarray(f1.t, np.float64))
    print(f"{a.config}: {e0.elapsed_time(e1) / a.frames:.3f} ms/frame (incl. one host sync), steps {res['steps']}, "
          f"inliers {res['inliers']}, |t - truth| {err * 1000:.2f} mm")


if __name__ == "__main__":
    main()
