"""Per-scene spatial index for the step kernel (host, init only).

The reference answers three geometry queries by brute force over every
segment of a world, every step (observation.py:91-100, rewards.py:86-94,
rewards.py:212-223).  The kernel keeps those exact float64 predicates and
only shrinks the set it evaluates them on, with candidate sets that are
provably supersets of every segment that can pass:

  * road context / edge boxes: a uniform grid of cell size >= 2 * (road
    radius + margin); a point's query square of half-width road_radius +
    margin touches at most 2 x 2 cells, and a per-cell bitmask over segment
    indices (bit q <=> midpoint q lies in the cell) OR-ed over those cells
    is a superset of all segments with d2 <= r^2, already in index order.
    Every edge box that a hull circle can touch has its midpoint within
    r + d + half_len + half_wid <= road_radius of the agent (checked here;
    otherwise the edge test falls back to the full scan).
  * nearest lane: per cell, the lane segments whose distance to the cell
    rectangle is <= the cell's upper bound ub(C) = min_s max_corner dist.
    The argmin of any point in the cell (and all its ties) is in that list,
    so an argmin over the list in ascending index order equals the full
    argmin, lowest index on ties.
Points outside the grid use the full scans.  Margins (1e-3 m on the grid,
1e-6 m on the lane bound) dominate every rounding error of the float64
geometry by many orders of magnitude.
"""

from __future__ import annotations

import math

import numpy as np

GRID_MARGIN = 4e-3      # m, query half-width = road_radius + GRID_MARGIN
LANE_MARGIN = 1e-6      # m, slack on the nearest-lane bound
HEADER_BYTES = 48       # f64 x0, y0, cell, half; i32 nx, ny, words, flags
FLAG_GRID = 1
FLAG_LANES = 2


def _pt_seg_dist(px, py, mx, my, ux, uy, hl):
    """Point-to-segment distance, the reference's (over, lat) form."""
    ex, ey = px - mx, py - my
    along = ex * ux + ey * uy
    lat = ux * ey - uy * ex
    over = np.maximum(np.abs(along) - hl, 0.0)
    return np.sqrt(over * over + lat * lat)


def _seg_rect_dist(ax, ay, bx, by, x0, y0, x1, y1):
    """Exact distance between segments [a, b] and axis-aligned rectangles
    (broadcast); 0 when they intersect."""
    def pt_rect(px, py):
        dx = np.maximum(np.maximum(x0 - px, 0.0), px - x1)
        dy = np.maximum(np.maximum(y0 - py, 0.0), py - y1)
        return np.sqrt(dx * dx + dy * dy)

    def pt_seg(px, py):
        vx, vy = bx - ax, by - ay
        L2 = vx * vx + vy * vy
        t = np.where(L2 > 0, ((px - ax) * vx + (py - ay) * vy) / np.where(L2 > 0, L2, 1.0), 0.0)
        t = np.clip(t, 0.0, 1.0)
        qx, qy = ax + t * vx - px, ay + t * vy - py
        return np.sqrt(qx * qx + qy * qy)

    d = np.minimum(pt_rect(ax, ay), pt_rect(bx, by))
    for cx, cy in ((x0, y0), (x1, y0), (x0, y1), (x1, y1)):
        d = np.minimum(d, pt_seg(cx, cy))

    def crosses(px, py, qx, qy):
        # segment [a,b] vs segment [p,q] proper/improper intersection
        def orient(ox, oy, sx, sy, tx, ty):
            return (sx - ox) * (ty - oy) - (sy - oy) * (tx - ox)
        o1 = orient(ax, ay, bx, by, px, py)
        o2 = orient(ax, ay, bx, by, qx, qy)
        o3 = orient(px, py, qx, qy, ax, ay)
        o4 = orient(px, py, qx, qy, bx, by)
        return (o1 * o2 <= 0) & (o3 * o4 <= 0)

    inside = ((ax >= x0) & (ax <= x1) & (ay >= y0) & (ay <= y1)) | crosses(x0, y0, x1, y0) | \
        crosses(x1, y0, x1, y1) | crosses(x1, y1, x0, y1) | crosses(x0, y1, x0, y0)
    return np.where(inside, 0.0, d)


def build_scene_index(mid, dirs, hl, hw, lane_index, edge_index, road_radius: float,
                      reach_max: float, max_cells: int = 4096, max_bytes: int = 96 * 1024):
    """Serialized index for one scene (little-endian bytes, 16-byte padded),
    or a header with flags = 0 when the scene does not qualify."""
    P = int(mid.shape[0])
    words = max(1, (P + 31) // 32)
    half = road_radius + GRID_MARGIN
    cell = 2.0 * half + 1e-3
    head = np.zeros(4, dtype=np.float64)
    ints = np.zeros(4, dtype=np.int32)
    if P == 0:
        return head.tobytes() + ints.tobytes()
    x0 = float(mid[:, 0].min()) - half
    y0 = float(mid[:, 1].min()) - half
    nx = int(math.floor((float(mid[:, 0].max()) + half - x0) / cell)) + 1
    ny = int(math.floor((float(mid[:, 1].max()) + half - y0) / cell)) + 1
    ncell = nx * ny
    head[:] = (x0, y0, cell, half)
    ints[:3] = (nx, ny, words)
    if ncell > max_cells:
        return head.tobytes() + ints.tobytes()

    cx = np.floor((mid[:, 0] - x0) / cell).astype(np.int64)
    cy = np.floor((mid[:, 1] - y0) / cell).astype(np.int64)
    bits = np.zeros((ncell, words), dtype=np.uint32)
    for q in range(P):
        bits[cy[q] * nx + cx[q], q >> 5] |= np.uint32(1 << (q & 31))
    edge_bits = np.zeros(words, dtype=np.uint32)
    for q in edge_index:
        edge_bits[q >> 5] |= np.uint32(1 << (int(q) & 31))
    flags = FLAG_GRID if reach_max <= road_radius else 0

    # nearest-lane candidate lists (indices into lane_index, ascending)
    starts = np.zeros(ncell + 1, dtype=np.int32)
    lists = []
    if len(lane_index):
        L = np.asarray(lane_index)
        lmx, lmy = mid[L, 0], mid[L, 1]
        lux, luy = dirs[L, 0], dirs[L, 1]
        lhl = hl[L]
        cid = np.arange(ncell)
        rx0 = x0 + cell * (cid % nx)          # cell c = cy * nx + cx
        ry0 = y0 + cell * (cid // nx)
        rx1, ry1 = rx0 + cell, ry0 + cell
        worst = np.zeros((ncell, len(L)))
        for qx, qy in ((rx0, ry0), (rx1, ry0), (rx0, ry1), (rx1, ry1)):
            worst = np.maximum(worst, _pt_seg_dist(qx[:, None], qy[:, None], lmx, lmy, lux, luy, lhl))
        ub = worst.min(axis=1)
        ax, ay = lmx - lhl * lux, lmy - lhl * luy
        bx, by = lmx + lhl * lux, lmy + lhl * luy
        lb = _seg_rect_dist(ax[None, :], ay[None, :], bx[None, :], by[None, :],
                            rx0[:, None], ry0[:, None], rx1[:, None], ry1[:, None])
        keep = lb <= (ub + LANE_MARGIN)[:, None]
        for c in range(ncell):
            ids = np.nonzero(keep[c])[0].astype(np.int32)
            lists.append(ids)
            starts[c + 1] = starts[c] + len(ids)
        flags |= FLAG_LANES
    lane_list = np.concatenate(lists).astype(np.int32) if lists else np.zeros(0, np.int32)
    ints[3] = flags
    out = head.tobytes() + ints.tobytes()
    for arr in (bits.reshape(-1), edge_bits, starts, lane_list):
        b = arr.tobytes()
        out += b + bytes((-len(b)) % 16)
    if len(out) > max_bytes:
        ints[3] = 0
        return head.tobytes() + ints.tobytes()
    return out
