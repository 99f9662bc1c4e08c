"""The spatial index only prunes: on random query points (on the map, on its
borders, far off it) the kernel's candidate sets, replayed here in numpy
exactly as the kernel reads the index, contain every segment the brute-force
reference predicates select, and the nearest-lane argmin over the candidate
list equals the full argmin (lowest index on ties)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.scenes import crossroads_scene, prepare_scene, straight_scene
from paper_2605_08528_b200.spatial import FLAG_GRID, FLAG_LANES, build_scene_index
from paper_2605_08528_b200.tables import SceneTable, _scene_table
from paper_2605_08528_b200.scenes import scene_segments


def parse(blob: bytes, P: int):
    hd = np.frombuffer(blob[:32], np.float64)
    nx, ny, words, flags = np.frombuffer(blob[32:48], np.int32)
    o = 48
    ncell = nx * ny

    def take(n, dt):
        nonlocal o
        a = np.frombuffer(blob[o:o + 4 * n], dt)
        o += (4 * n + 15) // 16 * 16
        return a

    bits = take(ncell * words, np.uint32).reshape(ncell, words)
    ebits = take(words, np.uint32)
    starts = take(ncell + 1, np.int32)
    lst = take(int(starts[-1]), np.int32)
    return dict(x0=hd[0], y0=hd[1], cell=hd[2], half=hd[3], nx=nx, ny=ny, words=words, flags=flags,
                bits=bits, ebits=ebits, starts=starts, lst=lst)


def superset(ix, px, py):
    inv = 1.0 / ix["cell"]
    cx0 = max(int(np.floor((px - ix["half"] - ix["x0"]) * inv)), 0)
    cx1 = min(int(np.floor((px + ix["half"] - ix["x0"]) * inv)), ix["nx"] - 1)
    cy0 = max(int(np.floor((py - ix["half"] - ix["y0"]) * inv)), 0)
    cy1 = min(int(np.floor((py + ix["half"] - ix["y0"]) * inv)), ix["ny"] - 1)
    out = set()
    if cx0 > cx1 or cy0 > cy1:
        return out
    for cy in range(cy0, cy1 + 1):
        for cx in range(cx0, cx1 + 1):
            for wd, word in enumerate(ix["bits"][cy * ix["nx"] + cx]):
                for b in range(32):
                    if int(word) >> b & 1:
                        out.add(wd * 32 + b)
    return out


def nearest(t: SceneTable, px, py, kks):
    best, bk = np.inf, None
    for kk in kks:
        q = t.lane_index[kk]
        ex, ey = px - t.midpoints[q, 0], py - t.midpoints[q, 1]
        ux, uy = t.directions[q]
        along = ex * ux + ey * uy
        lat = ux * ey - uy * ex
        over = max(abs(along) - t.half_lengths[q], 0.0)
        d2 = over * over + lat * lat
        if d2 < best:
            best, bk = d2, kk
    return bk


SCENES = [prepare_scene(straight_scene(agent_count=16, agent_gap=8.0, lane_offsets=(0.0, 4.0, -4.0))),
          prepare_scene(crossroads_scene(agent_count=16))]


@pytest.mark.parametrize("scene", SCENES, ids=["straight", "crossroads"])
def test_index_candidates_are_supersets(scene):
    t = _scene_table(scene_segments(scene))
    blob = build_scene_index(t.midpoints, t.directions, t.half_lengths, t.half_widths,
                             t.lane_index, t.edge_index, 10.0, 4.0)
    ix = parse(blob, t.num_segments)
    assert ix["flags"] & FLAG_GRID and ix["flags"] & FLAG_LANES
    g = np.random.Generator(np.random.Philox(7))
    pts = np.concatenate([g.uniform(-100, 100, (1500, 2)), g.uniform(-130, 130, (300, 2)),
                          t.midpoints + g.normal(0, 5, t.midpoints.shape)])
    edge = set(int(q) for q in t.edge_index)
    for px, py in pts:
        dx = t.midpoints[:, 0] - px
        dy = t.midpoints[:, 1] - py
        near = set(np.nonzero(dx * dx + dy * dy <= 100.0)[0].tolist())
        sup = superset(ix, px, py)
        assert near <= sup
        # edge boxes reachable by a hull (r + d + half_len + half_wid <= 4 m)
        reach = set(q for q in edge if np.hypot(dx[q], dy[q]) <= 4.0)
        assert reach <= sup
        fx = np.floor((px - ix["x0"]) / ix["cell"])
        fy = np.floor((py - ix["y0"]) / ix["cell"])
        if 0 <= fx < ix["nx"] and 0 <= fy < ix["ny"]:
            c = int(fy) * ix["nx"] + int(fx)
            cand = ix["lst"][ix["starts"][c]:ix["starts"][c + 1]]
            assert list(cand) == sorted(cand)
            assert nearest(t, px, py, cand) == nearest(t, px, py, range(len(t.lane_index)))


def test_index_disabled_when_boxes_outreach_the_grid():
    scene = SCENES[0]
    t = _scene_table(scene_segments(scene))
    blob = build_scene_index(t.midpoints, t.directions, t.half_lengths, t.half_widths,
                             t.lane_index, t.edge_index, 10.0, 10.5)
    assert not parse(blob, t.num_segments)["flags"] & FLAG_GRID


def test_default_pool_indexes_build():
    inp = C.build_inputs(C.RootConfig())
    assert inp.worlds.scene_tables is not None
