"""Per-scene spatial index for the step kernel (host, init only).

The reference answers three geometry queries by brute force over every
segment of a world, every step (observation.py:91-100, rewards.py:86-94,
rewards.py:212-223).  The kernel keeps those exact float64 predicates and
only shrinks the set it evaluates them on, with candidate sets that are
provably supersets of every segment that can pass:

  * road context / edge boxes: a uniform grid (cell = half / 2, half =
    road radius + margin); per cell, the ascending list of segments whose
    midpoint lies within `half` of the cell rectangle.  For any point in the
    cell it is a superset of the segments with d2 <= r^2, in index order.
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
HEADER_BYTES = 64       # f64 x0, y0, cell, half; i32 nx, ny, words, flags, 4 aux offsets
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


def _pt_rect_dist(px, py, x0, y0, x1, y1):
    dx = np.maximum(np.maximum(x0 - px, 0.0), px - x1)
    dy = np.maximum(np.maximum(y0 - py, 0.0), py - y1)
    return np.sqrt(dx * dx + dy * dy)


def _csr_u16(keep: np.ndarray):
    starts = np.zeros(keep.shape[0] + 1, dtype=np.int32)
    starts[1:] = np.cumsum(keep.sum(axis=1))
    rows, cols = np.nonzero(keep)          # row-major: per cell ascending index
    return starts, cols.astype(np.uint16)


def _pad16(b: bytes) -> bytes:
    return b + bytes((-len(b)) % 16)


def build_scene_index(mid, dirs, hl, hw, lane_index, edge_index, road_radius: float,
                      reach_max: float, cells_per_radius: int = 2, max_cells: int = 1 << 16):
    """Index of one scene: (header, aux).

    ``header`` (64 bytes) rides in the shared-memory scene blob:
    f64 x0, y0, cell, half; i32 nx, ny, words, flags; i32 byte offsets in aux
    of road_list, lane_start, lane_list, edge_bits.  ``aux`` stays in global
    memory (read through L1): i32 road_start[ncell+1], u16 road_list[] (segment
    index | is-edge << 15),
    i32 lane_start[ncell+1], u16 lane_list[], u32 edge_bits[words].
    Cell c = cy * nx + cx covers [x0 + cell*cx, +cell) x [y0 + cell*cy, +cell).
    """
    P = int(mid.shape[0])
    words = max(1, (P + 31) // 32)
    half = road_radius + GRID_MARGIN
    cell = half / cells_per_radius
    head = np.zeros(4, dtype=np.float64)
    ints = np.zeros(8, dtype=np.int32)
    if P == 0 or P > 32767:
        return head.tobytes() + ints.tobytes(), b""
    x0 = float(mid[:, 0].min()) - half
    y0 = float(mid[:, 1].min()) - half
    nx = int(math.floor((float(mid[:, 0].max()) + half - x0) / cell)) + 1
    ny = int(math.floor((float(mid[:, 1].max()) + half - y0) / cell)) + 1
    ncell = nx * ny
    head[:] = (x0, y0, cell, half)
    ints[:3] = (nx, ny, words)
    if ncell > max_cells:
        return head.tobytes() + ints.tobytes(), b""
    cid = np.arange(ncell)
    rx0 = x0 + cell * (cid % nx)
    ry0 = y0 + cell * (cid // nx)
    rx1, ry1 = rx0 + cell, ry0 + cell

    # road / edge-box superset: segments whose midpoint is within `half` of the cell
    near = _pt_rect_dist(mid[None, :, 0], mid[None, :, 1], rx0[:, None], ry0[:, None],
                         rx1[:, None], ry1[:, None]) <= half
    road_start, road_list = _csr_u16(near)
    flags = FLAG_GRID if reach_max <= road_radius else 0

    # nearest-lane candidates: lanes within ub(C) = min_s max_corner dist of the cell
    lane_start = np.zeros(ncell + 1, dtype=np.int32)
    lane_list = np.zeros(0, dtype=np.uint16)
    if len(lane_index):
        L = np.asarray(lane_index)
        lmx, lmy = mid[L, 0], mid[L, 1]
        lux, luy = dirs[L, 0], dirs[L, 1]
        lhl = hl[L]
        worst = np.zeros((ncell, len(L)))
        for qx, qy in ((rx0, ry0), (rx1, ry0), (rx0, ry1), (rx1, ry1)):
            worst = np.maximum(worst, _pt_seg_dist(qx[:, None], qy[:, None], lmx, lmy, lux, luy, lhl))
        ub = worst.min(axis=1)
        ax, ay = lmx - lhl * lux, lmy - lhl * luy
        bx, by = lmx + lhl * lux, lmy + lhl * luy
        lb = _seg_rect_dist(ax[None, :], ay[None, :], bx[None, :], by[None, :],
                            rx0[:, None], ry0[:, None], rx1[:, None], ry1[:, None])
        lane_start, lane_list = _csr_u16(lb <= (ub + LANE_MARGIN)[:, None])
        flags |= FLAG_LANES
    edge_bits = np.zeros(words, dtype=np.uint32)
    for q in edge_index:
        edge_bits[int(q) >> 5] |= np.uint32(1 << (int(q) & 31))
    # the road list carries the edge flag in bit 15 (segment index < 32768): the
    # scan gets "is this candidate a road edge" with the index, no dependent load
    is_edge = np.zeros(P, dtype=bool)
    is_edge[np.asarray(edge_index, dtype=np.int64)] = True
    road_list = road_list | (is_edge[road_list].astype(np.uint16) << np.uint16(15))

    aux = b""
    offs = []
    for arr in (road_start, road_list, lane_start, lane_list, edge_bits):
        offs.append(len(aux))
        aux += _pad16(arr.tobytes())
    ints[3] = flags
    ints[4:8] = offs[1:]
    return head.tobytes() + ints.tobytes(), aux
