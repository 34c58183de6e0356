"""Host-side control of the mapping step: the refinement round schedule and view selection.

PAPER.md P:157 "Gaussian optimization is launched every 10 frames, with 20 iterations performed
each time"; P:129 keyframes by camera motion (delta_angle, delta_move = 30 deg, 0.3 m),
n_global random keyframes + n_local evenly spaced recent frames (values not given; reading
R-VIEWS: 4 + 2); P:138 the selected views are raycast once per round and cached.
Reading R-VIEW: iteration i of a round renders the single view view[i mod V] (Table 2, P:237:
4000 iterations over 2000 frames = 2 per frame).  This module holds no arithmetic of the
rendering or fusion; it is plain bookkeeping (pure Python, tested on CPU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DELTA_K = 10
ITERATIONS = 20
DELTA_ANGLE_DEG = 30.0
DELTA_MOVE_M = 0.3
N_GLOBAL = 4        # R-VIEWS
N_LOCAL = 2         # R-VIEWS


def is_round_frame(k: int, delta_k: int = DELTA_K) -> bool:
    """Rounds run on frames k = 0, delta_k, 2 delta_k, ... (frame 0 included)."""
    return k % delta_k == 0


def round_frames(n_frames: int, delta_k: int = DELTA_K) -> list[int]:
    return [k for k in range(n_frames) if is_round_frame(k, delta_k)]


def local_views(interval: list[int], n_local: int = N_LOCAL) -> list[int]:
    """n_local frames evenly spread over the interval, ending at its last frame
    (10 frames, n_local = 2 -> interval positions 4 and 9)."""
    L = len(interval)
    if L == 0:
        return []
    n = min(n_local, L)
    return [interval[(j + 1) * L // n - 1] for j in range(n)]


def rotation_angle_deg(Ra: np.ndarray, Rb: np.ndarray) -> float:
    Rr = np.asarray(Ra, np.float64).T @ np.asarray(Rb, np.float64)
    c = (np.trace(Rr) - 1.0) / 2.0
    return math.degrees(math.acos(max(-1.0, min(1.0, c))))


@dataclass
class KeyframeSelector:
    """a frame becomes a keyframe if its rotation relative to the last keyframe exceeds
    delta_angle or its translation exceeds delta_move (frame 0 is the first keyframe)."""
    delta_angle_deg: float = DELTA_ANGLE_DEG
    delta_move_m: float = DELTA_MOVE_M
    keyframes: list = field(default_factory=list)   # frame ids
    _last: tuple | None = None

    def offer(self, k: int, R, t) -> bool:
        if self._last is None:
            add = True
        else:
            Rl, tl = self._last
            add = (rotation_angle_deg(Rl, R) > self.delta_angle_deg
                   or float(np.linalg.norm(np.asarray(t, np.float64) - np.asarray(tl, np.float64))) > self.delta_move_m)
        if add:
            self.keyframes.append(k)
            self._last = (np.asarray(R, np.float64), np.asarray(t, np.float64))
        return add


def select_views(keyframes: list[int], interval: list[int], rng: np.random.Generator,
                 n_global: int = N_GLOBAL, n_local: int = N_LOCAL) -> list[int]:
    """n_global keyframes sampled without replacement (all if fewer) + n_local local frames.
    Global views are drawn from keyframes outside the current interval when possible."""
    loc = local_views(interval, n_local)
    pool = [k for k in keyframes if k not in loc]
    g = sorted(rng.choice(pool, size=min(n_global, len(pool)), replace=False).tolist()) if pool else []
    return g + loc


def view_for_iteration(i: int, n_views: int) -> int:
    """Reading R-VIEW: iteration i renders view i mod V."""
    return i % n_views
