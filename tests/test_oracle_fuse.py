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
    """with w = 0 the update gives s = min(1, eta/mu) (no averaging).  Checked against
    the fp64 closed form (Z0 - z)/mu of a fronto-parallel plane, independent of the oracle's
    fp32 evaluation order (fp32 rounding of voxel position, depth and sample: <= 5e-6)."""
    c = cam()
    Z0 = 0.30
    depth, rgba = const_frame(c, Z0)
    v = O.Volume()
    v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba)
    co, ts, cw = v.blocks()
    P = voxel_world(co)
    # on the optical axis column of voxels (x = y = 0) the pixel is the principal point area
    sel = (np.abs(P[..., 0]) < 1e-9) & (np.abs(P[..., 1]) < 1e-9) & (cw[..., 3] == 1)
    assert sel.sum() >= 5
    z = P[..., 2][sel]
    expect = np.minimum(1.0, (Z0 - z) / MU)
    assert np.any(expect < 0) and np.any((expect > 0) & (expect < 1)) and np.any(expect == 1.0)
    assert np.max(np.abs(ts[sel] - expect)) <= 5e-6


def _plane_frames_pin(c, depths, rgbs, w_max=100):
    """Fuse fronto-parallel planes at the given depths (identity pose) and return, per voxel,
    (tsdf, rgbw, world z, clear mask): voxels away from the pixel-rounding boundaries that
    project inside the image, away from every frame's -mu decision boundary."""
    v = O.Volume(w_max=w_max)
    for Z, rgb in zip(depths, rgbs):
        d, col = const_frame(c, Z, rgb)
        v.fuse(c, np.eye(3), np.zeros(3), d, 1e4, col)
    co, ts, cw = v.blocks()
    P = voxel_world(co)
    z = P[..., 2]
    u = c.fx * P[..., 0] / np.where(z > 0, z, 1) + c.cx
    vv = c.fy * P[..., 1] / np.where(z > 0, z, 1) + c.cy
    ui, vi = np.floor(u + 0.5), np.floor(vv + 0.5)
    inside = (z > 0) & (ui >= 0) & (ui <= c.width - 1) & (vi >= 0) & (vi <= c.height - 1) \
        & (np.abs(u + 0.5 - np.round(u + 0.5)) > 1e-3) & (np.abs(vv + 0.5 - np.round(vv + 0.5)) > 1e-3)
    clear = inside.copy()
    for Z in depths:
        clear &= np.abs((Z - z) + MU) > 1e-4
    return ts, cw, z, clear


def test_tsdf_is_the_weighted_mean_of_the_samples():
    """P:60 / P:106 "standard SDF fusion" (reading R-INT): after frames at DISTINCT depths the
    voxel's tsdf is the mean of the samples s_k = min(1, (Z_k - z)/mu) of the frames that
    updated it (eta_k >= -mu), w = their number; a voxel no frame updated keeps tsdf 1, w 0.
    fp64 closed form; an update rule that ignores the weight (e.g. (tsdf + s)/2) fails it."""
    c = cam()
    depths = (0.30, 0.315, 0.33)
    ts, cw, z, clear = _plane_frames_pin(c, depths, [(9, 9, 9)] * 3)
    S = np.stack([np.minimum(1.0, (Z - z) / MU) for Z in depths])           # (3, n, 512)
    upd = np.stack([(Z - z) >= -MU for Z in depths])
    n_upd = upd.sum(0)
    mean = np.where(n_upd > 0, (S * upd).sum(0) / np.maximum(n_upd, 1), 1.0)
    w = cw[..., 3]
    assert np.all(w[clear] == n_upd[clear])
    for k in (1, 2, 3):
        sel = clear & (n_upd == k)
        assert sel.sum() >= 20, (k, sel.sum())
        assert np.max(np.abs(ts[sel] - mean[sel])) <= 5e-6, k
    # voxels whose samples differ across frames (not all clamped to 1): the mean is informative
    informative = clear & (n_upd == 3) & (np.ptp(np.where(upd, S, 0), axis=0) > 0.1)
    assert informative.sum() >= 20
    assert np.all(ts[clear & (n_upd == 0)] == 1.0)


def test_weight_cap_running_mean_closed_form():
    """R-WMAX with distinct samples: w_max = 2, three frames.  The third update weighs the
    stored mean by the capped weight: tsdf = (2*mean(s1, s2) + s3)/3, w = 2."""
    c = cam()
    depths = (0.30, 0.31, 0.32)
    ts, cw, z, clear = _plane_frames_pin(c, depths, [(9, 9, 9)] * 3, w_max=2)
    s = [np.minimum(1.0, (Z - z) / MU) for Z in depths]
    all3 = clear & np.all(np.stack([(Z - z) >= -MU for Z in depths]), 0)
    assert all3.sum() >= 20
    exp = (2.0 * (s[0] + s[1]) / 2.0 + s[2]) / 3.0
    assert np.max(np.abs(ts[all3] - exp[all3])) <= 5e-6
    assert np.all(cw[..., 3][all3] == 2)


def _round_half_up_mean(values):
    """the exact rational running mean of u8 observations, rounded half up at each update
    (R-INT), computed with exact fractions: floor(mean + 1/2) -- never the integer formula."""
    from fractions import Fraction
    c, w = 0, 0
    for x in values:
        m = Fraction(c * w + x, w + 1)
        c = int(np.floor(m + Fraction(1, 2)))
        w += 1
    return c


@pytest.mark.parametrize("seq", [(51, 154), (10, 20, 32), (200, 3, 101, 7), (255, 0), (0, 255)])
def test_colour_mean_rounds_half_up(seq):
    """R-INT colour: the per-channel running mean is the exact rational mean rounded half up
    (51, 154 -> 102.5 -> 103; 10, 20, 32 -> 15 then 62/3 + ... -> 21).  A truncating mean
    fails the .5 and the w = 2 cases."""
    c = cam()
    v = O.Volume()
    for x in seq:
        d, col = const_frame(c, 0.5, (x, x, x))
        v.fuse(c, np.eye(3), np.zeros(3), d, 1e4, col)
    _, _, cw = v.blocks()
    seen = cw[..., 3] == len(seq)
    assert seen.sum() > 100
    assert np.all(cw[..., :3][seen] == _round_half_up_mean(seq))


def test_budget_overflow_flag():
    """exceeding the block budget is a hard error carrying the budget."""
    c = cam()
    depth, rgba = const_frame(c, 0.3)
    v = O.Volume(budget=10)
    assert v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba) == 2
    assert v.overflow and v.n_blocks > 10
