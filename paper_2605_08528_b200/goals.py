"""Goal resampling along the start lane (``eval.random_goals``).

Restates drivegrid config.py:222-278: for every valid agent, the nearest lane
polyline to its start, a target arc length drawn on Philox stream (seed, 4)
(uniform in [goal_min_m, goal_max_m], or exactly goal_min_m when the range is
empty), tried forward then backward along the lane; agents whose lane is too
short keep their goal.
"""

from __future__ import annotations

import numpy as np


def polyline_arc_point(points: np.ndarray, start_arc: float, distance: float):
    seg = np.diff(points[:, :2], axis=0)
    seg_len = np.sqrt((seg ** 2).sum(axis=1))
    cum = np.concatenate([[0.0], np.cumsum(seg_len)])
    target = start_arc + distance
    if target < 0.0 or target > cum[-1]:
        return None
    i = min(int(np.searchsorted(cum, target, side="right") - 1), len(seg_len) - 1)
    frac = (target - cum[i]) / seg_len[i] if seg_len[i] > 0 else 0.0
    return points[i, :2] + frac * seg[i]


def resample_goal(start_xy, scene, min_m: float, max_m: float, rng):
    lanes = scene.lane_polylines()
    if not lanes:
        return None
    best = None
    for poly in lanes:
        pts = poly.points[:, :2]
        d2 = ((pts - start_xy) ** 2).sum(axis=1)
        i = int(np.argmin(d2))
        if best is None or d2[i] < best[0]:
            seg = np.diff(pts, axis=0)
            cum = np.concatenate([[0.0], np.cumsum(np.sqrt((seg ** 2).sum(axis=1)))])
            best = (d2[i], poly, cum[i])
    _, poly, start_arc = best
    dist = min_m if min_m == max_m else rng.uniform(min_m, max_m)
    for sign in (1.0, -1.0):
        pt = polyline_arc_point(poly.points, start_arc, sign * dist)
        if pt is not None:
            return pt
    return None


def resample_goals(goal_xy, start_xy, valid, grid_offsets, pool, assignment, cfg):
    """New goals on the nearest lane, Philox stream (seed, 4); returns a copy."""
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([cfg.seed, 4])))
    goal_xy = goal_xy.copy()
    W, M = valid.shape
    for w in range(W):
        off = grid_offsets[w]
        for m in range(M):
            if not valid[w, m]:
                continue
            g = resample_goal(start_xy[w, m] - off, pool[assignment[w]], cfg.eval.goal_min_m,
                              cfg.eval.goal_max_m, rng)
            if g is not None:
                goal_xy[w, m] = g + off
    return goal_xy


def resample_engine_goals(engine, pool, assignment, cfg) -> None:
    engine.set_goals(resample_goals(engine.goal_xy, engine.start_xy, engine.valid,
                                    engine.worlds.grid_offsets, pool, assignment, cfg))
