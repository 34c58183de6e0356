"""Pins of the oracle's allocation (O2) and integration (O3) against closed forms, invariants,
worked examples and a brute-force exact band enumeration -- never against itself.
PAPER.md P:60 (voxel contents), P:106 (fusion into a global hash table); readings R-BAND,
R-INT, R-MU, R-WMAX in DESIGN.md §3."""
import numpy as np
import pytest

import oracle as O
from tests.refimpl import random_rotation

VOX, MU = 0.005, 0.02


def cam(w=64, h=48, f=60.0):
    return O.Camera(f, f, (w - 1) / 2, (h - 1) / 2, w, h)


def const_frame(c, z, rgb=(200, 100, 50), scale=1e4):
    depth = np.full((c.height, c.width), int(round(z * scale)), np.uint16)
    rgba = np.zeros((c.height, c.width, 4), np.uint8)
    rgba[..., :3] = rgb
    rgba[..., 3] = 255
    return depth, rgba


def voxel_world(coords):
    """world position of every voxel of the exported blocks: (n,512,3), index i+8j+64k."""
    k, j, i = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")
    loc = np.stack([i.reshape(-1), j.reshape(-1), k.reshape(-1)], axis=1)  # (512,3) ordered i fastest
    g = coords[:, None, :] * 8 + loc[None]
    return g.astype(np.float64) * np.float64(np.float32(VOX))


def test_empty_depth_allocates_nothing():
    """an empty depth map gives 0 new blocks."""
    c = cam()
    v = O.Volume()
    depth = np.zeros((c.height, c.width), np.uint16)
    rgba = np.zeros((c.height, c.width, 4), np.uint8)
    assert v.fuse(c, np.eye(3), np.zeros(3), depth, 1000.0, rgba) == 0
    assert v.n_blocks == 0


def test_fronto_parallel_plane_closed_form_with_general_pose():
    """O3 closed form: for a plane fronto-parallel to the camera at depth Z0 the
    depth image is constant, so every voxel with camera z <= Z0 + mu that projects into the
    image gets tsdf = min(1, (Z0 - z)/mu) after one frame, colour = the plane colour exactly,
    w = 1; voxels farther than mu behind stay untouched.  A non-identity pose pins the
    world->camera convention X = R^T (P - t) (R-POSE): a transposed R breaks it."""
    rng = np.random.default_rng(1)
    c = cam(96, 72, 80.0)
    R = random_rotation(rng)
    t = np.array([0.3, -0.2, 0.5], np.float32)
    Z0 = 0.8
    depth, rgba = const_frame(c, Z0)
    v = O.Volume()
    assert v.fuse(c, R, t, depth, 1e4, rgba) == 0
    coords, tsdf, rgbw = v.blocks()
    assert len(coords) > 20
    P = voxel_world(coords)
    X = (P - t.astype(np.float64)) @ R.astype(np.float64)  # R^T (P - t), row form
    z = X[..., 2]
    u = c.fx * X[..., 0] / z + c.cx
    vv = c.fy * X[..., 1] / z + c.cy
    ui, vi = np.floor(u + 0.5), np.floor(vv + 0.5)
    inside = (z > 0) & (ui >= 0) & (ui <= c.width - 1) & (vi >= 0) & (vi <= c.height - 1)
    eta = Z0 - z
    w = rgbw[..., 3]
    margin = 1e-4  # stay away from the pixel-rounding and -mu decision boundaries
    clear_in = inside & (eta >= -MU + margin) & (np.abs(u + 0.5 - np.round(u + 0.5)) > 1e-3) \
        & (np.abs(vv + 0.5 - np.round(vv + 0.5)) > 1e-3)
    clear_out = (~inside & (np.abs(u + 0.5 - np.round(u + 0.5)) > 1e-3)) | (eta < -MU - margin)
    assert clear_in.sum() > 1000
    assert np.all(w[clear_in] == 1)
    assert np.all(w[clear_out & (z > 0)] == 0)
    exp = np.minimum(1.0, eta / MU)
    assert np.max(np.abs(tsdf[clear_in] - exp[clear_in])) <= 1e-5
    assert np.all(rgbw[clear_in][:, :3] == np.array([200, 100, 50]))
    assert np.all(tsdf[w == 0] == 1.0)


def test_band_blocks_match_exact_dda():
    """O2 against a brute-force traversal: every block met by the exact (fp64) band segment
    [X(1-mu/|X|), X(1+mu/|X|)] of some pixel is allocated, and every allocated block lies within
    one block of such a segment (R-BAND)."""
    rng = np.random.default_rng(2)
    c = cam(40, 30, 40.0)
    R = random_rotation(rng)
    t = np.array([-0.4, 0.1, 0.2], np.float32)
    zmap = rng.uniform(0.5, 2.5, size=(c.height, c.width))
    depth = np.round(zmap * 1000).astype(np.uint16)
    depth[rng.random(depth.shape) < 0.1] = 0
    rgba = np.zeros((c.height, c.width, 4), np.uint8)
    v = O.Volume()
    v.fuse(c, R, t, depth, 1000.0, rgba)
    got = {tuple(b) for b in v.visible()}
    assert got == {tuple(b) for b in v.blocks()[0]}  # first frame: allocated == visible
    bs = 8 * VOX
    exact = set()
    near_any = set()
    Rd, td = R.astype(np.float64), t.astype(np.float64)
    for y in range(c.height):
        for x in range(c.width):
            d = depth[y, x] / 1000.0
            if not (0.1 <= d <= 10):
                continue
            X = np.array([(x - c.cx) / c.fx * d, (y - c.cy) / c.fy * d, d])
            n = np.linalg.norm(X)
            A = Rd @ (X * (1 - MU / n)) + td
            B = Rd @ (X * (1 + MU / n)) + td
            # dense sampling of the segment (1/2000 block spacing) approximates exact DDA
            for s in np.linspace(0, 1, 400):
                Q = A + (B - A) * s
                exact.add(tuple(np.floor(Q / bs).astype(int)))
                for dq in ((1e-6, 0, 0), (-1e-6, 0, 0), (0, 1e-6, 0), (0, -1e-6, 0), (0, 0, 1e-6), (0, 0, -1e-6)):
                    near_any.add(tuple(np.floor((Q + np.array(dq)) / bs).astype(int)))
    # R-BAND allocates the boxes spanned by consecutive samples: a superset of the exact
    # traversal, never farther than one block (Chebyshev) from a block the segment meets
    assert exact <= got, f"{len(exact - got)} blocks met by a band segment were not allocated"
    ex = np.array(sorted(near_any))
    for b in got - near_any:
        assert np.min(np.max(np.abs(ex - np.array(b)), axis=1)) <= 1
    assert len(got) <= 1.6 * len(exact)


def test_idempotent_refusion_and_weight_cap():
    """fusing the same frame again allocates no new block; N identical
    frames leave tsdf (within fp32 rounding of the running mean) and colour unchanged with
    w = min(N, w_max)."""
    c = cam()
    depth, rgba = const_frame(c, 0.5, (10, 20, 30))
    v = O.Volume(w_max=3)
    v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba)
    co1, ts1, cw1 = v.blocks()
    for k in range(5):
        v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba)
        co, ts, cw = v.blocks()
        assert np.array_equal(co, co1)
        touched = cw1[..., 3] > 0
        assert np.all(cw[..., 3][touched] == min(k + 2, 3))
        assert np.all(cw[..., :3][touched] == np.array([10, 20, 30]))
        assert np.max(np.abs(ts[touched] - ts1[touched])) <= 2e-7
        assert np.all(cw[..., 3][~touched] == 0)


def test_colour_running_mean_worked_example():
    """two observations of colours 0.2 and 0.6 fuse to 0.4.  In u8: 51 then 153 ->
    (51*1 + 153 + 1) div 2 = 102 = 0.4*255 exactly (R-INT)."""
    c = cam()
    d1, c1 = const_frame(c, 0.5, (51, 51, 51))
    d2, c2 = const_frame(c, 0.5, (153, 153, 153))
    v = O.Volume()
    v.fuse(c, np.eye(3), np.zeros(3), d1, 1e4, c1)
    v.fuse(c, np.eye(3), np.zeros(3), d2, 1e4, c2)
    _, _, cw = v.blocks()
    seen = cw[..., 3] == 2
    assert seen.sum() > 100
    assert np.all(cw[..., :3][seen] == 102)


def test_first_observation_copies_sample():
    """with w = 0 the update gives exactly s = min(1, eta/mu) (no averaging)."""
    c = cam()
    depth, rgba = const_frame(c, 0.30)
    v = O.Volume()
    v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba)
    co, ts, cw = v.blocks()
    P = voxel_world(co)
    # on the optical axis column of voxels (x = y = 0) the pixel is the principal point area
    sel = (np.abs(P[..., 0]) < 1e-9) & (np.abs(P[..., 1]) < 1e-9) & (cw[..., 3] == 1)
    assert sel.sum() >= 5
    z = P[..., 2][sel].astype(np.float32)
    # the sample s of DESIGN.md §4.2: d = raw * fl(1/scale), s = min(1, (d - z) * fl(1/mu))
    d = np.float32(3000) * (np.float32(1.0) / np.float32(1e4))
    expect = np.minimum(np.float32(1.0), (d - z) * (np.float32(1.0) / np.float32(MU)))
    assert np.max(np.abs(ts[sel] - expect)) == 0.0


def test_budget_overflow_flag():
    """exceeding the block budget is a hard error carrying the budget."""
    c = cam()
    depth, rgba = const_frame(c, 0.3)
    v = O.Volume(budget=10)
    assert v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba) == 2
    assert v.overflow and v.n_blocks > 10
