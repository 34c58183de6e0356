"""Shared set-up for the -m gpu parity tests: the same seeded inputs (gps_synth) go to the CUDA
path (through the C ABI) and to the CPU oracle; nothing the CUDA path produces ever feeds the
oracle."""
from __future__ import annotations

import numpy as np
import torch

import gps_synth as S
import oracle as O


def cams(cfg):
    import paper_2509_11574_b200 as G
    return (G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height),
            O.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height))


def frames(cfg, n, start=0):
    return S.make_frames(cfg, n, start=start, device="cpu")


def to_dev(fr):
    return fr.depth.cuda(), fr.rgba.cuda()


def gpu_volume(cfg, **kw):
    import paper_2509_11574_b200 as G
    args = dict(voxel_size=cfg.voxel_size, w_max=100, depth_min=0.1, depth_max=10.0,
                max_blocks=cfg.max_blocks, hash_slots=cfg.hash_slots)
    args.update(kw)
    return G.Volume(**args)


def oracle_volume(cfg, **kw):
    args = dict(voxel_size=cfg.voxel_size, mu=4 * cfg.voxel_size, w_max=100, depth_min=0.1, depth_max=10.0)
    args.update(kw)
    return O.Volume(**args)


def fuse_both(cfg, frs, gvol=None, ovol=None):
    gcam, ocam = cams(cfg)
    gvol = gvol or gpu_volume(cfg)
    ovol = ovol or oracle_volume(cfg)
    for fr in frs:
        d, c = to_dev(fr)
        gvol.fuse(gcam, fr.R, fr.t, d, cfg.depth_scale, c)
        ovol.fuse(ocam, fr.R, fr.t, fr.depth.numpy().view(np.uint16), cfg.depth_scale, fr.rgba.numpy())
    torch.cuda.synchronize()
    return gvol, ovol


def sorted_blocks(coords, vox=None):
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    return coords[order], (None if vox is None else vox[order])


def rel_err(a, b, floor):
    return np.abs(a - b) / np.maximum(np.abs(b), floor)
