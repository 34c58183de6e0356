"""Pins of the oracle raycast (O4; "marched through the SDF voxels to find
the zero crossing ... linearly interpolating the colors of the eight neighboring voxels ...
projecting V onto the image plane"; reading R-RAY) against closed forms and analytic scenes."""
import numpy as np

import oracle as O
from tests.refimpl import random_rotation


def cam(w=48, h=36, f=45.0):
    return O.Camera(f, f, (w - 1) / 2, (h - 1) / 2, w, h)


def test_fronto_parallel_plane_depth_is_exact():
    """Within +-mu the fused field of a fronto-parallel plane is exactly linear in camera z;
    trilinear interpolation and linear refinement are exact on linear fields, so
    D_t = Z0 up to the fp32 rounding of the stored tsdf (~1e-9 m) on every interior pixel.
    C_t equals the uniform plane colour."""
    c = cam()
    Z0 = 0.4
    depth = np.full((c.height, c.width), 4000, np.uint16)
    rgba = np.zeros((c.height, c.width, 4), np.uint8)
    rgba[..., :3] = (30, 160, 90)
    v = O.Volume()
    v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba)
    D, col, V, _ = v.raycast(c, np.eye(3), np.zeros(3))
    D = D.reshape(c.height, c.width)
    interior = np.zeros_like(D, bool)
    interior[3:-3, 3:-3] = True
    assert np.all(D[interior] > 0)
    assert np.max(np.abs(D[interior] - Z0)) < 1e-6
    col = col.reshape(c.height, c.width, 3)
    assert np.max(np.abs(col[interior] - np.array([30, 160, 90]) / 255.0)) < 1e-9
    # V* lies on the plane and on the pixel's ray: its projection is the pixel itself
    V = V.reshape(c.height, c.width, 3)
    ys, xs = np.nonzero(interior)
    Vi = V[ys, xs]
    assert np.max(np.abs(Vi[:, 2] - Z0)) < 1e-6
    assert np.max(np.abs(c.fx * Vi[:, 0] / Vi[:, 2] + c.cx - xs)) < 1e-6


def test_plane_from_general_pose():
    """Same closed form with a rotated, translated camera (pins the camera->world ray)."""
    rng = np.random.default_rng(5)
    c = cam()
    R = random_rotation(rng)
    t = np.array([0.2, 0.5, -0.3], np.float32)
    depth = np.full((c.height, c.width), 6000, np.uint16)
    rgba = np.full((c.height, c.width, 4), 128, np.uint8)
    v = O.Volume()
    v.fuse(c, R, t, depth, 1e4, rgba)
    D, _, _, _ = v.raycast(c, R, t)
    D = D.reshape(c.height, c.width)[4:-4, 4:-4]
    assert np.all(D > 0)
    assert np.max(np.abs(D - 0.6)) < 2e-6


def test_unallocated_space_is_a_miss():
    """a ray through unallocated space misses: D_t = 0 and C_t = 0."""
    c = cam()
    depth = np.full((c.height, c.width), 4000, np.uint16)
    rgba = np.full((c.height, c.width, 4), 200, np.uint8)
    v = O.Volume()
    v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba)
    R = np.array([[-1, 0, 0], [0, 1, 0], [0, 0, -1]], np.float32)  # looking backwards
    D, col, _, _ = v.raycast(c, R, np.zeros(3))
    assert np.all(D == 0) and np.all(col == 0)
    # an empty volume misses everywhere
    D, col, _, _ = O.Volume().raycast(c, np.eye(3), np.zeros(3))
    assert np.all(D == 0) and np.all(col == 0)


def sphere_depth(c, R, t, centre, r):
    ys, xs = np.mgrid[0:c.height, 0:c.width]
    dc = np.stack([(xs - c.cx) / c.fx, (ys - c.cy) / c.fy, np.ones_like(xs, float)], -1)
    dn = dc / np.linalg.norm(dc, axis=-1, keepdims=True)
    dw = dn @ R.astype(np.float64).T
    oc = t.astype(np.float64) - centre
    b = dw @ oc
    disc = b * b - (oc @ oc - r * r)
    tt = -b - np.sqrt(np.maximum(disc, 0))
    z = np.where(disc > 0, tt * dn[..., 2], 0.0)
    return z


def test_sphere_rmse_below_voxel():
    """S:163 / AC5: fused analytic sphere (r = 0.5 m seen from ~2 m) raycast depth has
    RMSE < voxel_size against the analytic depth over sampled pixels hit by both.  The camera
    resolves the voxel size (pixel footprint 4 mm at 2 m) so the projective distance is sharp."""
    c = O.Camera(500.0, 500.0, 159.5, 119.5, 320, 240)
    centre = np.array([0.0, 0.0, 0.0])
    r = 0.5
    v = O.Volume()
    poses = []
    for k, yaw in enumerate(np.linspace(-0.3, 0.3, 4)):
        eye = np.array([2.0 * np.sin(yaw), 0.1 * k - 0.15, -2.0 * np.cos(yaw)])
        f = -eye / np.linalg.norm(eye)
        x = np.cross(f, [0, 1.0, 0])
        x /= np.linalg.norm(x)
        y = np.cross(f, x)
        R = np.stack([x, y, f], 1).astype(np.float32)
        t = eye.astype(np.float32)
        poses.append((R, t))
        z = sphere_depth(c, R, t, centre, r)
        depth = np.round(z * 1e4).astype(np.uint16)
        rgba = np.full((c.height, c.width, 4), 180, np.uint8)
        v.fuse(c, R, t, depth, 1e4, rgba)
    R, t = poses[1]
    rng = np.random.default_rng(0)
    pix = np.stack([rng.integers(0, c.width, 3000), rng.integers(0, c.height, 3000)], 1).astype(np.int32)
    D, col, _, _ = v.raycast(c, R, t, pix)
    z = sphere_depth(c, R, t, centre, r)[pix[:, 1], pix[:, 0]]
    both = (D > 0) & (z > 0)
    assert both.sum() > 0.98 * (z > 0).sum()
    # projective TSDF fattens silhouettes slightly: false hits only as a thin rim
    assert ((D > 0) & (z == 0)).sum() <= 0.01 * (z > 0).sum()
    rmse = np.sqrt(np.mean((D[both] - z[both]) ** 2))
    assert rmse < 0.005, rmse
    assert np.max(np.abs(col[both] - 180 / 255.0)) < 1e-9


def test_negative_region_entered_from_unobserved_space_is_a_miss():
    """R-RAY "invalid predecessor => miss" ("find the zero crossing": a crossing needs a
    valid positive sample before the first valid non-positive one).  A plane fused from the
    front (Z0 = 0.4 m) and raycast from BEHIND it: the rays come from unobserved voxels (w = 0,
    invalid) straight into the negative band behind the surface, so no +/- crossing exists and
    every pixel is a miss.  Seen from the front the same volume is hit everywhere."""
    c = cam()
    Z0 = 0.4
    depth = np.full((c.height, c.width), 4000, np.uint16)
    rgba = np.full((c.height, c.width, 4), 77, np.uint8)
    v = O.Volume()
    v.fuse(c, np.eye(3), np.zeros(3), depth, 1e4, rgba)
    Rb = np.array([[-1, 0, 0], [0, 1, 0], [0, 0, -1]], np.float32)   # looking along -z
    tb = np.array([0.0, 0.0, 0.8], np.float32)                       # 0.4 m behind the plane
    D, col, _, margin = v.raycast(c, Rb, tb)
    assert np.all(D == 0) and np.all(col == 0)
    # the rays do reach valid, negative samples (so the miss is the predecessor rule, not range)
    assert np.sum(np.isfinite(margin)) > 0.5 * D.size
    Df, _, _, _ = v.raycast(c, np.eye(3), np.zeros(3))
    assert np.mean(Df > 0) > 0.8
