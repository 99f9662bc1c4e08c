"""CPU oracle of the episode safety metrics -- TEST INFRASTRUCTURE ONLY.

Float64 numpy restatement of the reference's per-step pairwise DRAC and the
episode aggregation (``/root/reference/pkg/src/drivegrid/metrics.py``).  Only
``tests/`` and ``bench.py``'s CPU legs may import it.  Pinned against the
reference's own outputs by ``tests/test_oracle_golden.py`` (fixture
``tests/golden/drac_wet.npz`` / ``drac_events.npz``, made by
``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import numpy as np

DRAC_THRESHOLD = 3.4          # metrics.py:21
CLEARANCE_FLOOR = 1e-2        # metrics.py:59-61
DIST_FLOOR = 1e-9             # metrics.py:50


def world_velocity(vx, vy, yaw):
    """metrics.py:104-107: body velocity rotated into the world frame."""
    c, s = np.cos(yaw), np.sin(yaw)
    return vx * c - vy * s, vx * s + vy * c


def pairwise_drac(px, py, yaw, vwx, vwy, r_hull, d_hull, alive):
    """Per-agent max DRAC against alive neighbours (metrics.py:33-62).

    For the ordered pair (i, j) of one world: d = p_j - p_i, u = v_j - v_i,
    closing = -(d.u)/max(|d|, 1e-9); clearance = min over the 3x3 hull-circle
    pairs of the centre distance minus (r_i + r_j); DRAC = closing^2 /
    (2 max(clearance, 1e-2)) where both agents are alive, i != j, closing > 0
    and clearance > 1e-2, else 0.  Returns max over j, shape (W, M)."""
    W, M = alive.shape
    if M < 2:
        return np.zeros((W, M))
    dx = px[:, None, :] - px[:, :, None]          # [w, i, j] = p_j - p_i
    dy = py[:, None, :] - py[:, :, None]
    dist = np.sqrt(dx * dx + dy * dy)
    ux = vwx[:, None, :] - vwx[:, :, None]
    uy = vwy[:, None, :] - vwy[:, :, None]
    closing = -(dx * ux + dy * uy) / np.maximum(dist, DIST_FLOOR)

    c, s = np.cos(yaw), np.sin(yaw)
    ox, oy = d_hull * c, d_hull * s               # offsets (-1, 0, +1) x (d cos, d sin)
    best = np.full((W, M, M), np.inf)
    for a in (-1.0, 0.0, 1.0):
        ax = px + a * ox
        ay = py + a * oy
        for b in (-1.0, 0.0, 1.0):
            bx = px + b * ox
            by = py + b * oy
            ex = ax[:, :, None] - bx[:, None, :]
            ey = ay[:, :, None] - by[:, None, :]
            best = np.minimum(best, np.sqrt(ex * ex + ey * ey))
    clearance = best - (r_hull[:, :, None] + r_hull[:, None, :])

    ok = alive[:, :, None] & alive[:, None, :] & ~np.eye(M, dtype=bool)[None]
    ok &= (closing > 0.0) & (clearance > CLEARANCE_FLOOR)
    val = np.where(ok, closing * closing / (2.0 * np.maximum(clearance, CLEARANCE_FLOOR)), 0.0)
    return val.max(axis=-1)


def drac_of_snapshot(state: dict, alive_pre, r_hull, d_hull):
    """pairwise_drac on one logged step (metrics.py:101-108): the post-physics,
    pre-park state snapshot with the alive mask from before the step."""
    vwx, vwy = world_velocity(state["v_x"], state["v_y"], state["yaw"])
    return pairwise_drac(state["x"], state["y"], state["yaw"], vwx, vwy, r_hull, d_hull,
                         np.asarray(alive_pre, dtype=bool))


def aggregate(goal_seen, coll_seen, max_drac, valid, threshold=DRAC_THRESHOLD) -> dict:
    """episode_metrics' reduction (metrics.py:110-125)."""
    valid = np.asarray(valid, dtype=bool)
    n = int(valid.sum())
    goals = int((goal_seen & valid).sum())
    colls = int((coll_seen & valid).sum())
    over = max_drac[valid & (max_drac > threshold)]
    return {"sr": goals / n if n else 0.0, "cr": colls / n if n else 0.0,
            "mean_max_drac": float(over.mean()) if over.size else 0.0,
            "valid_agents": n, "goals": goals, "collisions": colls}
