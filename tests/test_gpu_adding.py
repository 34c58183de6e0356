"""GPU parity of Gaussian adding and removal (gps_vertex_normals, gps_add_gaussians_sync,
gps_remove_gaussians_sync) against oracle/adding.py on the same seeded
stand-in inputs (gps_synth.adding_stage_inputs; no CUDA output feeds the oracle).

Bars: the Eq. 6 mask, the sampled set and its row-major order, and the removal set are
integer results decided in fp32 on both sides -- bit-exact; normals within 1e-4; positions and
colours of new Gaussians within 1e-6; kNN scales within 1e-4 relative; survivors of a removal bitwise equal to the kept rows."""
import numpy as np
import pytest
import torch

import gps_synth as S
from oracle import adding as OA

pytestmark = pytest.mark.gpu


def _inputs(cfg_name="cfg2", start=0):
    cfg = S.get_config(cfg_name)
    fr = S.make_frames(cfg, 1, start=start)[0]
    return cfg, fr, S.adding_stage_inputs(cfg, fr, seed=start)


def _gpu_normals(G, cfg, fr, x):
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    Dt, V = torch.from_numpy(x["Dt"]).cuda(), torch.from_numpy(x["V"]).cuda()
    return cam, Dt, V, G.vertex_normals(cam, fr.R, fr.t, Dt, V)


def test_vertex_normals_match_oracle():
    import paper_2509_11574_b200 as G
    cfg, fr, x = _inputs()
    cam, Dt, V, N = _gpu_normals(G, cfg, fr, x)
    on = OA.vertex_normals(x["V"].astype(np.float64), x["Dt"], fr.t)
    gn = N.cpu().numpy()
    assert np.array_equal(np.abs(gn).sum(-1) > 0, np.abs(on).sum(-1) > 0)
    assert np.max(np.abs(gn - on)) <= 1e-4
    assert (np.abs(on).sum(-1) > 0).mean() > 0.5


@pytest.mark.parametrize("cfg_name,deg", [("cfg1", 3), ("cfg2", 3), ("cfg2", 0)])
def test_add_gaussians_matches_oracle(cfg_name, deg):
    import paper_2509_11574_b200 as G
    cfg, fr, x = _inputs(cfg_name)
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    Dt, V = torch.from_numpy(x["Dt"]).cuda(), torch.from_numpy(x["V"]).cuda()
    # both sides take the same seeded normal map: the scene's analytic normals (misses zeroed)
    nin = fr.normal.numpy().astype(np.float32).copy()
    nin[x["Dt"] == 0] = 0.0
    N = torch.from_numpy(nin).cuda()
    on = nin.astype(np.float64)
    n0 = 50
    rng = np.random.default_rng(1)
    g0 = S.random_gaussians(n0, deg, rng)
    g = G.Gaussians.from_dict(g0, capacity=n0 + cfg.width * cfg.height)
    st = G.AdamState(g)
    st.m.xyz.fill_(1.0)
    st.step = 7
    cfgA = G.AddConfig(seed=123)
    added, cand = G.add_gaussians(g, st, cam, Dt, V, N, torch.from_numpy(x["Cstar"]).cuda(),
                                  torch.from_numpy(x["WG"]).cuda(), torch.from_numpy(x["target"]).cuda().contiguous(),
                                  cfgA)
    M = OA.add_mask(x["Cstar"], x["WG"], x["Dt"], on, x["target"])
    keep = OA.sample_keep(cfg.width * cfg.height, seed=123).reshape(M.shape)
    sel = M & keep
    assert added == cand == int(sel.sum()) > 20
    assert g.n == n0 + added and st.m.n == g.n and st.step == 7
    Vm = x["V"].astype(np.float64).reshape(-1, 3)[np.flatnonzero(M.reshape(-1))]
    midx = np.cumsum(M.reshape(-1)) - 1
    q = midx[np.flatnonzero(sel.reshape(-1))]
    s1, tie = OA.knn_scale(Vm, q)
    ref = OA.init_gaussians(x["V"].astype(np.float64), on, x["target"], sel, s1, deg)
    got = g.to_numpy()
    new = slice(n0, g.n)
    assert np.array_equal(got["xyz"][:n0], g0["xyz"].astype(np.float32))  # old rows untouched
    assert np.allclose(got["xyz"][new], ref["xyz"], atol=1e-6)
    assert np.allclose(got["sh"][new], ref["sh"], atol=2e-6)
    assert np.allclose(got["opacity_raw"][new], ref["opacity_raw"], atol=1e-7)
    assert np.allclose(got["rot"][new], ref["rot"], atol=1e-4)
    # the RMS of the 3 smallest distances does not depend on which of several equidistant 3rd
    # neighbours is taken, so ties (regular pixel grids on planes) need no exclusion
    gs = np.exp(got["log_scale"][new].astype(np.float64))
    rs = np.exp(ref["log_scale"])
    assert np.all(np.abs(gs - rs) <= 1e-4 * rs)
    assert (rs[:, 0] < 0.1).mean() > 0.5  # most scales come from real neighbours, not the cap
    # the new rows' Adam moments are fresh, the old rows' kept
    m = st.m.to_numpy()
    assert np.all(m["xyz"][new] == 0) and np.all(m["xyz"][:n0] == 1.0)


def test_add_respects_capacity():
    import paper_2509_11574_b200 as G
    cfg, fr, x = _inputs("cfg1")
    cam = G.Camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)
    Dt, V = torch.from_numpy(x["Dt"]).cuda(), torch.from_numpy(x["V"]).cuda()
    N = torch.from_numpy(fr.normal.numpy().astype(np.float32)).cuda()
    g = G.Gaussians.from_dict(S.random_gaussians(10, 1, np.random.default_rng(2)), capacity=15)
    st = G.AdamState(g)
    added, cand = G.add_gaussians(g, st, cam, Dt, V, N, torch.from_numpy(x["Cstar"]).cuda(),
                                  torch.from_numpy(x["WG"]).cuda(), torch.from_numpy(x["target"]).cuda().contiguous())
    assert added == 5 and cand > 5 and g.n == 15


def test_remove_gaussians_matches_oracle():
    import paper_2509_11574_b200 as G
    rng = np.random.default_rng(4)
    n = 5000
    gd = S.random_gaussians(n, 3, rng)
    # spread opacities and scales across the Eq. 8 thresholds
    gd["opacity_raw"] = rng.uniform(-7, 3, n).astype(np.float32)
    gd["log_scale"] = np.log(rng.uniform(0.001, 0.15, (n, 3))).astype(np.float32)
    g = G.Gaussians.from_dict(gd)
    st = G.AdamState(g)
    mm = {k: rng.normal(size=getattr(g, k).shape).astype(np.float32) for k in ("xyz", "log_scale", "rot", "opacity_raw", "sh")}
    for k, v in mm.items():
        getattr(st.m, k).copy_(torch.from_numpy(v))
        getattr(st.v, k).copy_(torch.from_numpy(np.abs(v)))
    removed = G.remove_gaussians(g, st)
    rm = OA.remove_mask(gd["opacity_raw"], gd["log_scale"])
    assert removed == int(rm.sum()) and 0.2 < rm.mean() < 0.9
    keep = ~rm
    got = g.to_numpy()
    for k in ("xyz", "log_scale", "rot", "opacity_raw", "sh"):
        assert np.array_equal(got[k], np.asarray(gd[k], np.float32)[keep]), k
        assert np.array_equal(st.m.to_numpy()[k], mm[k][keep]), k
        assert np.array_equal(st.v.to_numpy()[k], np.abs(mm[k])[keep]), k
