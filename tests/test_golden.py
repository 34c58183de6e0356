"""The paper's printed constants (tests/golden/paper_constants.json, each with its PAPER.md
line) are the defaults of the oracle and of the product's Python configs."""
import json
import os

import numpy as np

import oracle as O

HERE = os.path.dirname(__file__)


def load(name):
    with open(os.path.join(HERE, "golden", name)) as f:
        return json.load(f)


def test_oracle_defaults_are_the_papers():
    g = load("paper_constants.json")
    a = O.AdamCfg()
    assert a.lr_xyz == g["lr_position"]["value"]
    assert a.lr_sh0 == g["lr_sh0"]["value"]
    assert a.lr_opacity == g["lr_alpha"]["value"]
    assert a.lr_scale == g["lr_scale"]["value"]
    assert a.lr_rot == g["lr_rotation"]["value"]
    assert a.lr_shrest == g["lr_sh_rest"]["value"]
    assert abs(O.RenderCfg().alpha_min - g["alpha_clamp"]["value"]) < 1e-15


def test_backprojection_convention_example():
    """fx = fy = 100, cx = cy = 50, pixel (60, 50), depth 2 -> (0.2, 0, 2.0), the pixel-
    centre convention R-PIX used by the oracle's allocation (X = ((u-cx)/fx d, (v-cy)/fy d, d))."""
    e = load("spec_worked_examples.json")["backproject"]
    u, v = e["pixel"]
    d = e["depth"]
    X = np.array([(u - e["cx"]) / e["fx"] * d, (v - e["cy"]) / e["fy"] * d, d])
    assert np.allclose(X, e["vertex"], atol=1e-12)
    # the oracle allocates the block holding that vertex for this single pixel
    c = O.Camera(e["fx"], e["fy"], e["cx"], e["cy"], 101, 101)
    depth = np.zeros((101, 101), np.uint16)
    depth[v, u] = 2000
    vol = O.Volume()
    vol.fuse(c, np.eye(3), np.zeros(3), depth, 1000.0, np.zeros((101, 101, 4), np.uint8))
    blocks = {tuple(b) for b in vol.visible()}
    centre = tuple(np.floor((X + np.array([1e-7, 1e-7, 1e-7])) / 0.04).astype(int))
    assert centre in blocks
