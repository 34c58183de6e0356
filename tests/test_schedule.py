"""Host logic of the round schedule: exact."""
import numpy as np

from paper_2509_11574_b200 import schedule as Sch
from tests.refimpl import rot_z


def test_rounds_every_delta_k_including_frame_0():
    """delta_k = 10 and 25 frames give rounds at frames 0, 10, 20."""
    assert Sch.round_frames(25) == [0, 10, 20]
    assert Sch.DELTA_K == 10 and Sch.ITERATIONS == 20


def test_even_local_selection():
    """a 10-frame interval with n_local = 2 selects interval positions 4 and 9."""
    interval = list(range(30, 40))
    assert Sch.local_views(interval, 2) == [34, 39]
    assert Sch.local_views([0], 2) == [0]


def test_keyframe_motion_rule():
    """keyframe when rotation > 30 deg or translation > 0.3 m vs the last one."""
    ks = Sch.KeyframeSelector()
    I = np.eye(3)
    assert ks.offer(0, I, [0, 0, 0])
    assert not ks.offer(1, I, [0.29, 0, 0])
    assert ks.offer(2, I, [0.31, 0, 0])
    assert not ks.offer(3, rot_z(np.radians(29)), [0.31, 0, 0])
    assert ks.offer(4, rot_z(np.radians(31)), [0.31, 0, 0])
    assert ks.keyframes == [0, 2, 4]


def test_view_selection_and_round_robin():
    rng = np.random.default_rng(0)
    v = Sch.select_views([0, 7, 15, 22, 31, 44], list(range(40, 50)), rng)
    assert v[-2:] == [44, 49] and len(v) == 6 and len(set(v)) == 6
    v2 = Sch.select_views([0, 7, 15, 22, 31, 44], list(range(40, 50)), np.random.default_rng(0))
    assert v == v2  # seeded
    assert [Sch.view_for_iteration(i, 6) for i in range(8)] == [0, 1, 2, 3, 4, 5, 0, 1]
    assert Sch.select_views([], [0], rng) == [0]
