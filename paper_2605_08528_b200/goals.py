"""Goal resampling along the start lane (``eval.random_goals``).

Behaviour of drivegrid config.py:222-278: every valid agent gets a new goal
on the lane polyline whose vertex lies nearest its (scene-local) start; the
travel distance is drawn from Philox stream (seed, 4) -- uniform in
[goal_min_m, goal_max_m], or exactly goal_min_m when the range is empty, one
draw per valid agent in (world, agent) order -- and is walked forward along
the lane from the nearest vertex's arc length, else backward; an agent whose
lane is too short either way keeps its goal.  Arithmetic (cumulative arc
lengths, the interpolation) is term for term the reference's, so the goals are
bit-identical (tests/test_oracle_golden.py, golden ``goals_random``).
"""

from __future__ import annotations

import numpy as np


def _arc_table(pts: np.ndarray):
    """(segment vectors, their lengths, cumulative arc length at each vertex)."""
    seg = np.diff(pts, axis=0)
    length = np.sqrt((seg ** 2).sum(axis=1))
    return seg, length, np.concatenate([[0.0], np.cumsum(length)])


def polyline_arc_point(points: np.ndarray, start_arc: float, distance: float):
    """The point ``distance`` metres of arc past ``start_arc`` (negative:
    before it), or None off either end of the polyline."""
    seg, length, arc = _arc_table(points[:, :2])
    target = start_arc + distance
    if not 0.0 <= target <= arc[-1]:
        return None
    k = min(int(np.searchsorted(arc, target, side="right")) - 1, len(length) - 1)
    along = (target - arc[k]) / length[k] if length[k] > 0 else 0.0
    return points[k, :2] + along * seg[k]


def _nearest_lane(start_xy, lanes):
    """(lane, arc length of its vertex nearest ``start_xy``); ties keep the
    earlier lane and, within a lane, the earlier vertex."""
    best_d2, pick = np.inf, None
    for lane in lanes:
        pts = lane.points[:, :2]
        d2 = ((pts - start_xy) ** 2).sum(axis=1)
        v = int(np.argmin(d2))
        if pick is None or d2[v] < best_d2:
            best_d2, pick = d2[v], (lane, _arc_table(pts)[2][v])
    return pick


def resample_goal(start_xy, scene, min_m: float, max_m: float, rng):
    """One agent's new goal (scene-local), or None (no lanes, or the lane is
    too short for the drawn distance in both directions)."""
    lanes = scene.lane_polylines()
    if not lanes:
        return None
    lane, arc0 = _nearest_lane(start_xy, lanes)
    reach = min_m if min_m == max_m else rng.uniform(min_m, max_m)
    ahead = polyline_arc_point(lane.points, arc0, reach)
    return ahead if ahead is not None else polyline_arc_point(lane.points, arc0, -reach)


def resample_goals(goal_xy, start_xy, valid, grid_offsets, pool, assignment, cfg):
    """New goals for every valid slot of a (W, M) batch; returns a copy."""
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([cfg.seed, 4])))
    out = np.array(goal_xy, dtype=np.float64, copy=True)
    for w, m in zip(*np.nonzero(valid)):          # row-major: (world, agent) order
        off = grid_offsets[w]
        g = resample_goal(start_xy[w, m] - off, pool[assignment[w]], cfg.eval.goal_min_m,
                          cfg.eval.goal_max_m, rng)
        if g is not None:
            out[w, m] = g + off
    return out


def resample_engine_goals(engine, pool, assignment, cfg) -> None:
    engine.set_goals(resample_goals(engine.goal_xy, engine.start_xy, engine.valid,
                                    engine.worlds.grid_offsets, pool, assignment, cfg))
