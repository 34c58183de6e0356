"""Tracked-trajectory error of the mapping pipeline on a cfg sequence, with the host pose read
every frame (eager) or only when needed (deferred, as bench.py runs it).  Diagnostic only.

    python tools/track_diag.py [--config cfg4] [--frames 120] [--history 60]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gps_synth as S  # noqa: E402
import paper_2509_11574_b200 as G  # noqa: E402
from paper_2509_11574_b200.pipeline import MappingPipeline  # noqa: E402


def run(cfg, frames, history, eager, n_g, watch=None, icp=None):
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    vol = G.Volume(voxel_size=cfg.voxel_size, max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots,
                   dense_bounds=S.scene_bounds(cfg))
    g = G.Gaussians.from_dict(S.make_gaussians(cfg, n=n_g))
    pipe = MappingPipeline(cam, g, vol, cfg.depth_scale, seed=0, track=True, icp_cfg=icp)
    for k, (d, c, R, t) in enumerate(frames):
        pipe.process_frame(k, d, c, R, t, refine=k >= history)
        if eager and watch and watch[0] <= k <= watch[1]:
            nz = (pipe.t_normal != 0).any(-1).float().mean().item()
            hit = (pipe.depth > 0).float().mean().item()
            dv = ((d.view(torch.int16).to(torch.int32) & 0xFFFF) > 0).float().mean().item()
            print(f"  after frame {k}: model normals {nz:.3f} raycast hits {hit:.3f} depth valid {dv:.3f} "
                  f"log {pipe.track_log[-1]['inliers'] if k else None}")
        if eager:
            pipe.last_pose
    pipe.join()
    pipe.last_pose  # reads back the pending poses
    torch.cuda.synchronize()
    err = [float(np.linalg.norm(pipe.poses[k][1].astype(np.float64) - np.asarray(frames[k][3], np.float64)))
           for k in range(len(frames))]
    return np.array(err), vol.stats()["n_blocks"], pipe.track_log


def bilateral(d_u16: torch.Tensor, scale: float, r=3, sig_s=4.5, sig_r=0.03) -> torch.Tensor:
    """Diagnostic-only depth pre-filter (KinectFusion-style bilateral), torch ops."""
    z = (d_u16.view(torch.int16).to(torch.int32) & 0xFFFF).to(torch.float32) / scale
    H, W = z.shape
    zp = torch.nn.functional.pad(z[None, None], (r, r, r, r))
    patches = torch.nn.functional.unfold(zp, 2 * r + 1).view((2 * r + 1) ** 2, H, W)
    yy, xx = torch.meshgrid(torch.arange(-r, r + 1), torch.arange(-r, r + 1), indexing="ij")
    ws = torch.exp(-(xx ** 2 + yy ** 2).float() / (2 * sig_s ** 2)).reshape(-1, 1, 1).to(z.device)
    wr = torch.exp(-((patches - z[None]) ** 2) / (2 * sig_r ** 2)) * (patches > 0)
    w = ws * wr
    out = (w * patches).sum(0) / w.sum(0).clamp_min(1e-12)
    out = torch.where(z > 0, out, torch.zeros_like(out))
    return torch.round(out * scale).to(torch.int32).to(torch.int16).contiguous()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--frames", type=int, default=120)
    ap.add_argument("--history", type=int, default=60)
    ap.add_argument("--gaussians", type=int, default=20000)
    ap.add_argument("--detail", type=int, default=0, help="print ICP records of this many frames before failure")
    ap.add_argument("--watch", type=int, nargs=2, default=None, help="print model-map stats for these frames")
    ap.add_argument("--angle", type=float, default=30.0)
    ap.add_argument("--filter", type=int, default=3, help="R-ICP-FILT radius (0 = off)")
    ap.add_argument("--dist", type=float, default=0.1)
    ap.add_argument("--prefilter", action="store_true", help="bilateral-filter the depth frames first")
    ap.add_argument("--clean", action="store_true", help="noise-free depth")
    ap.add_argument("--both", action="store_true", help="also the deferred read-back")
    a = ap.parse_args()
    cfg = S.get_config(a.config, **({"noise": "none", "dropout": 0.0} if a.clean else {}))
    scene = S.make_scene(cfg)
    dc = S.pixel_rays(cfg, "cuda")
    poses = S.trajectory(cfg, a.frames)
    frames = []
    for k in range(a.frames):
        fr = S.render_frame(cfg, scene, *poses[k], k=k, device="cuda", dc=dc)
        dep = bilateral(fr.depth, cfg.depth_scale) if a.prefilter else fr.depth.contiguous()
        frames.append((dep, fr.rgba.contiguous(), fr.R, fr.t))
    for eager in (True, False):
        icp = G.IcpConfig(angle_max_deg=a.angle, dist_max=a.dist, filter_radius=a.filter)
        err, nb, log = run(cfg, frames, a.history, eager, a.gaussians, watch=a.watch, icp=icp)
        bad = np.nonzero(err > 0.02)[0]
        print(f"eager={eager}: max err {err.max():.4f} m, rmse {np.sqrt(np.mean(err ** 2)):.4f}, blocks {nb}, "
              f"first frame > 2 cm: {bad[0] if len(bad) else None}")
        print("  err every 10th frame:", np.round(err[::10], 4).tolist())
        if a.detail and (len(bad) or a.detail < 0):
            f0, f1 = (1, len(frames)) if a.detail < 0 else (max(1, bad[0] - a.detail), min(len(frames), bad[0] + 3))
            for f in range(f0, f1):
                r = log[f - 1]  # frame f's ICP (frame 0 is not tracked)
                dR = np.asarray(frames[f][2], np.float64) @ np.asarray(frames[f - 1][2], np.float64).T
                ang = np.degrees(np.arccos(np.clip((np.trace(dR) - 1) / 2, -1, 1)))
                mv = np.linalg.norm(np.asarray(frames[f][3], np.float64) - np.asarray(frames[f - 1][3], np.float64))
                print(f"  frame {f}: err {err[f]:.4f} true step {mv * 1000:.1f} mm {ang:.2f} deg | steps {r['steps']} "
                      f"inl {r['inlier_frac']:.3f} n {r['inliers']} conv {r['converged']} piv {r['pivot_ratio']:.2e} degen {r['degenerate']} energy {r['energy']:.3g}")
        if not a.both:
            break


if __name__ == "__main__":
    main()
