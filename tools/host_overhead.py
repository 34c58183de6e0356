#!/usr/bin/env python3
"""Is the mapping step host-bound?  Times the host side of enqueuing K steps (fuse + raycast per
frame, a refinement round per step, two streams) against the device time of the same steps.

    python tools/host_overhead.py [--steps 10]
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
from paper_2509_11574_b200.pipeline import MappingPipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--history", type=int, default=30)
    ap.add_argument("--cprofile", action="store_true", help="cProfile the enqueue loop (host hot spots)")
    args = ap.parse_args()
    cfg = S.get_config("cfg4")
    scene = S.make_scene(cfg)
    dc = S.pixel_rays(cfg, "cuda")
    n = args.history + 10 * (args.steps + 2)
    poses = S.trajectory(cfg, n)
    frames = [S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc) for k in range(n)]
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots,
                   dense_bounds=S.scene_bounds(cfg))
    g = G.Gaussians.from_dict(S.make_gaussians(cfg))
    pipe = MappingPipeline(cam, g, vol, cfg.depth_scale)
    k = 0
    for _ in range(args.history):
        f = frames[k]
        pipe.process_frame(k, f.depth, f.rgba, f.R, f.t, refine=False)
        k += 1
    while (k + 9) % 10 != 0:
        f = frames[k]
        pipe.process_frame(k, f.depth, f.rgba, f.R, f.t, refine=False)
        k += 1
    for _ in range(10):  # warm-up step
        f = frames[k]
        pipe.process_frame(k, f.depth, f.rgba, f.R, f.t)
        k += 1
    pipe.join()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    prof = None
    if args.cprofile:
        import cProfile
        prof = cProfile.Profile()
        prof.enable()
    h0 = time.perf_counter()
    for _ in range(10 * args.steps):
        f = frames[k]
        pipe.process_frame(k, f.depth, f.rgba, f.R, f.t)
        k += 1
    h1 = time.perf_counter()
    if prof is not None:
        prof.disable()
        import pstats
        pstats.Stats(prof).sort_stats("tottime").print_stats(25)
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    print(f"host enqueue {1000 * (h1 - h0) / args.steps:.3f} ms/step, device {e0.elapsed_time(e1) / args.steps:.3f} "
          f"ms/step, wall {1000 * (h2 - h0) / args.steps:.3f} ms/step")


if __name__ == "__main__":
    main()
