#!/usr/bin/env python3
"""Per-tile list lengths of one refine iteration on a steady-state cfg4 state (diagnostics for
the blend/backward load balance): entries per tile before and after the depth pre-cull.

    python tools/tile_stats.py [--history 60] [--tile 16]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gps_synth as S  # noqa: E402
import paper_2509_11574_b200 as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--history", type=int, default=60)
    ap.add_argument("--tile", type=int, default=16)
    args = ap.parse_args()
    cfg = S.get_config("cfg4")
    scene = S.make_scene(cfg)
    dc = S.pixel_rays(cfg, "cuda")
    poses = S.trajectory(cfg, args.history + 1)
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots,
                   dense_bounds=S.scene_bounds(cfg))
    f = None
    for k in range(args.history):
        f = S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc)
        vol.fuse(cam, f.R, f.t, f.depth, cfg.depth_scale, f.rgba)
    g = G.Gaussians.from_dict(S.make_gaussians(cfg))
    st = G.AdamState(g)
    ras = G.Rasterizer(g.n, cam, G.RenderConfig(tile=args.tile))
    D, C, _ = vol.raycast(cam, f.R, f.t)
    view = G.View(cam, f.R, f.t, D, C, f.rgba)
    ras.refine_step(g, st, [view])
    torch.cuda.synchronize()
    vals, ranges = ras.lists()
    tiles_x = -(-cfg.width // args.tile)
    n_full = np.diff(np.append(ranges[:, 0].astype(np.int64), len(vals)))
    n_eff = ranges[:, 1].astype(np.int64) - ranges[:, 0].astype(np.int64)
    for name, n in (("listed", n_full), ("after pre-cull", n_eff)):
        q = np.percentile(n, [50, 90, 99, 99.9, 100])
        top = np.sort(n)[::-1]
        print(f"{name}: total {n.sum()} mean {n.mean():.1f} p50/p90/p99/p99.9/max {q.astype(int).tolist()} "
              f"top10 {top[:10].tolist()} share of top 1% tiles {top[:max(1, len(n) // 100)].sum() / max(n.sum(), 1):.3f}")
    t = int(np.argmax(n_eff))
    print("heaviest tile", t, "at", (t % tiles_x, t // tiles_x), "n", n_full[t], "n_eff", n_eff[t])
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", "tile_stats.npz"), n_full=n_full, n_eff=n_eff)


if __name__ == "__main__":
    main()
