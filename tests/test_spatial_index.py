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


def parse(head: bytes, aux: bytes):
    hd = np.frombuffer(head[:32], np.float64)
    nx, ny, words, flags, o_rl, o_ls, o_ll, o_eb = np.frombuffer(head[32:64], np.int32)
    ncell = nx * ny
    rs = np.frombuffer(aux[:4 * (ncell + 1)], np.int32)
    rl_raw = np.frombuffer(aux[o_rl:o_rl + 2 * int(rs[-1])], np.uint16)
    rl = rl_raw & np.uint16(0x7FFF)
    ls = np.frombuffer(aux[o_ls:o_ls + 4 * (ncell + 1)], np.int32)
    ll = np.frombuffer(aux[o_ll:o_ll + 2 * int(ls[-1])], np.uint16)
    return dict(x0=hd[0], y0=hd[1], cell=hd[2], half=hd[3], nx=nx, ny=ny, words=words, flags=flags,
                road_start=rs, road_list=rl, road_edge=(rl_raw >> 15).astype(bool), lane_start=ls, lane_list=ll)


def cell_of(ix, px, py):
    inv = 1.0 / ix["cell"]
    fx = np.floor((px - ix["x0"]) * inv)
    fy = np.floor((py - ix["y0"]) * inv)
    if 0 <= fx < ix["nx"] and 0 <= fy < ix["ny"]:
        return int(fy) * ix["nx"] + int(fx)
    return -1


def superset(ix, px, py):
    c = cell_of(ix, px, py)
    if c < 0:
        return set()
    return set(ix["road_list"][ix["road_start"][c]:ix["road_start"][c + 1]].tolist())


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
    ix = parse(*build_scene_index(t.midpoints, t.directions, t.half_lengths, t.half_widths,
                                  t.lane_index, t.edge_index, 10.0, 4.0))
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
        c = cell_of(ix, px, py)
        if c >= 0:
            rl = ix["road_list"][ix["road_start"][c]:ix["road_start"][c + 1]]
            assert list(rl) == sorted(rl)
            cand = ix["lane_list"][ix["lane_start"][c]:ix["lane_start"][c + 1]]
            assert list(cand) == sorted(cand)
            assert nearest(t, px, py, cand) == nearest(t, px, py, range(len(t.lane_index)))


def test_index_disabled_when_boxes_outreach_the_grid():
    scene = SCENES[0]
    t = _scene_table(scene_segments(scene))
    head, aux = build_scene_index(t.midpoints, t.directions, t.half_lengths, t.half_widths,
                                  t.lane_index, t.edge_index, 10.0, 10.5)
    assert not parse(head, aux)["flags"] & FLAG_GRID


def test_default_pool_indexes_build():
    inp = C.build_inputs(C.RootConfig())
    assert inp.worlds.scene_tables is not None


def test_road_list_edge_flags():
    """bit 15 of every road-list entry == the segment is a road edge."""
    for scene in SCENES:
        t = _scene_table(scene_segments(scene))
        head, aux = build_scene_index(t.midpoints, t.directions, t.half_lengths, t.half_widths,
                                      t.lane_index, t.edge_index, 10.0, 4.0)
        ix = parse(head, aux)
        edge = set(int(q) for q in t.edge_index)
        assert ix["road_list"].size
        for q, e in zip(ix["road_list"], ix["road_edge"]):
            assert bool(e) == (int(q) in edge)
