#!/usr/bin/env python3
"""Drive the hot calls on a steady-state cfg4 state for targeted profiling (ncu -k regex:...).

    python tools/kernel_bench.py [--history 60] [--iters 3] [--only fuse|raycast|refine|all]
Prints per-call device time (CUDA events) so the plain run doubles as a quick timing check.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gps_synth as S  # noqa: E402
import paper_2509_11574_b200 as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--history", type=int, default=60)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--only", default="all")
    ap.add_argument("--gaussians", type=int, default=0)
    ap.add_argument("--sort-free", action="store_true")
    args = ap.parse_args()
    cfg = S.get_config(args.config)
    scene = S.make_scene(cfg)
    dc = S.pixel_rays(cfg, "cuda")
    poses = S.trajectory(cfg, args.history + args.iters + 1)
    frames = [S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc) for k in range(len(poses))]
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots,
                   dense_bounds=None if os.environ.get("GPS_NO_GRID") else S.scene_bounds(cfg))
    for k in range(args.history):
        f = frames[k]
        vol.fuse(cam, f.R, f.t, f.depth, cfg.depth_scale, f.rgba)
    gd = S.make_gaussians(cfg, n=args.gaussians or None)
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    ras = G.Rasterizer(g.n, cam, G.RenderConfig(sort_free=int(args.sort_free)))
    D = torch.empty((cfg.height, cfg.width), device="cuda")
    C = torch.empty((cfg.height, cfg.width, 3), device="cuda")
    f = frames[args.history - 1]
    vol.raycast(cam, f.R, f.t, D, C)
    view = G.View(cam, f.R, f.t, D, C, f.rgba)
    torch.cuda.synchronize()
    times = {"fuse": [], "raycast": [], "refine": []}
    for i in range(args.iters):
        f = frames[args.history + i]
        for name, fn in (("fuse", lambda: vol.fuse(cam, f.R, f.t, f.depth, cfg.depth_scale, f.rgba)),
                         ("raycast", lambda: vol.raycast(cam, f.R, f.t, D, C)),
                         ("refine", lambda: ras.refine_step(g, st, [view]))):
            if args.only not in ("all", name):
                continue
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            times[name].append(e0.elapsed_time(e1))
    print({k: [round(x, 4) for x in v] for k, v in times.items() if v})
    print("hits", float((D > 0).float().mean()), "stats", vol.stats(), ras.stats())


if __name__ == "__main__":
    main()
