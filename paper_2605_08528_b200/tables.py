"""Host-built engine tables: spawn table, per-world friction, per-scene segment tables.

Built once per engine from the world batch.  The device engine uploads them;
the CPU oracle (tests only) consumes the very same arrays, so parity runs
compare two steppers over identical inputs.

Reference anchors (``/root/reference/pkg/src/drivegrid/engine.py``):
  * geometry in global coordinates, lane/edge compaction  176-186, 234-253
  * mu_eff = min(mu_static, ground)                        188-190
  * spawn table, parked empty slots                        192-227
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .friction import ground_material
from .params import (LANE_CENTER_CODES, OFFSTAGE_X, ROAD_EDGE_CODES, STATE_FIELDS,
                     SimConfig, VehicleParams)
from .scenes import SegmentArray, WorldBatch, filter_agents


def circle_layout(length, width, wheelbase: float):
    """Three-circle hull radius and offset (observation.py:44-48)."""
    r = np.maximum(0.45, 0.55 * np.asarray(width, dtype=np.float64))
    d = np.minimum(wheelbase / 2.0,
                   np.maximum(0.0, np.asarray(length, dtype=np.float64) / 2.0 - 0.8 * r))
    return r, d


def lane_mask_of(type_codes, seg_mask):
    return seg_mask & ((type_codes == LANE_CENTER_CODES[0]) | (type_codes == LANE_CENTER_CODES[1]))


def edge_mask_of(type_codes, seg_mask):
    return seg_mask & ((type_codes == ROAD_EDGE_CODES[0]) | (type_codes == ROAD_EDGE_CODES[1]))


@dataclass
class SceneTable:
    """One scene's segments in scene-local coordinates + lane/edge index lists."""

    midpoints: np.ndarray     # (P, 2) f64
    directions: np.ndarray    # (P, 2) f64
    type_codes: np.ndarray    # (P,) i32
    half_lengths: np.ndarray  # (P,) f64
    half_widths: np.ndarray   # (P,) f64
    lane_index: np.ndarray    # (K_lane,) i32, ascending segment index
    edge_index: np.ndarray    # (K_edge,) i32, ascending segment index

    @property
    def num_segments(self) -> int:
        return int(self.midpoints.shape[0])


@dataclass
class EngineTables:
    W: int
    M: int
    grid_offsets: np.ndarray   # (W, 2)
    scene_of_world: np.ndarray  # (W,) i64
    scenes: list                # [SceneTable]
    mu_eff: np.ndarray          # (W,)
    weather: np.ndarray         # (W, 4)
    valid: np.ndarray           # (W, M) bool
    start_xy: np.ndarray        # (W, M, 2) global
    goal_xy: np.ndarray         # (W, M, 2) global
    start_yaw: np.ndarray       # (W, M)
    length: np.ndarray          # (W, M)
    width: np.ndarray           # (W, M)
    r_hull: np.ndarray          # (W, M)
    d_hull: np.ndarray          # (W, M)
    state0: dict                # field -> (W, M) f64, initial state


def _scene_table(seg: SegmentArray) -> SceneTable:
    codes = np.asarray(seg.type_codes, dtype=np.int32)
    ok = np.ones(len(codes), dtype=bool)
    return SceneTable(
        np.ascontiguousarray(seg.midpoints, dtype=np.float64).reshape(-1, 2),
        np.ascontiguousarray(seg.directions, dtype=np.float64).reshape(-1, 2),
        codes,
        np.ascontiguousarray(seg.half_lengths, dtype=np.float64),
        np.ascontiguousarray(seg.half_widths, dtype=np.float64),
        np.nonzero(lane_mask_of(codes, ok))[0].astype(np.int32),
        np.nonzero(edge_mask_of(codes, ok))[0].astype(np.int32))


def scene_tables_of(worlds: WorldBatch):
    """Per-scene tables and the world->table map.  Batches imported from the
    binary format carry no scene tables; their worlds are de-duplicated by
    content instead."""
    if worlds.scene_tables is not None and worlds.scene_index is not None:
        return [_scene_table(s) for s in worlds.scene_tables], np.asarray(worlds.scene_index)
    tables, index, seen = [], np.zeros(worlds.num_worlds, dtype=np.int64), {}
    for w in range(worlds.num_worlds):
        n = int(worlds.mask[w].sum())
        key = b"".join(a[w, :n].tobytes() for a in (worlds.midpoints, worlds.directions,
                                                    worlds.type_codes, worlds.half_lengths,
                                                    worlds.half_widths))
        if key not in seen:
            seen[key] = len(tables)
            tables.append(_scene_table(SegmentArray(worlds.midpoints[w, :n], worlds.directions[w, :n],
                                                    worlds.type_codes[w, :n], worlds.half_lengths[w, :n],
                                                    worlds.half_widths[w, :n])))
        index[w] = seen[key]
    return tables, index


def world_friction(frictions, params: VehicleParams):
    """Per-world mu_eff = min(mu_static, dry ground) and the weather token
    (engine.py:188-190)."""
    ground_mu, _ = ground_material(1.0, params.f_lon_dry, params.f_lat_dry)
    mu_eff = np.array([min(f.mu_static, ground_mu) for f in frictions], dtype=np.float64)
    weather = np.stack([f.weather_token for f in frictions], axis=0).astype(np.float64)
    return mu_eff, weather


def build_tables(worlds: WorldBatch, scenes, assignment, frictions, config: SimConfig,
                 params: VehicleParams) -> EngineTables:
    W, M = config.num_envs, config.num_agents
    if worlds.num_worlds != W:
        raise ValueError(f"world batch has {worlds.num_worlds} worlds, config wants {W}")
    if len(frictions) != W:
        raise ValueError("need one friction assignment per world")
    mu_eff, weather = world_friction(frictions, params)

    state = {k: np.zeros((W, M)) for k in STATE_FIELDS}
    state["brake_sign_front"][:] = 1.0
    state["brake_sign_rear"][:] = 1.0
    valid = np.zeros((W, M), dtype=bool)
    start_xy = np.zeros((W, M, 2))
    goal_xy = np.zeros((W, M, 2))
    start_yaw = np.zeros((W, M))
    length = np.full((W, M), 4.0)
    width = np.full((W, M), 2.0)
    offs = worlds.grid_offsets
    spawn_cache = {}
    for w in range(W):
        s = int(assignment[w])
        if s not in spawn_cache:
            spawn_cache[s] = filter_agents(scenes[s], bbox_half=config.bbox_half,
                                           goal_radius=config.goal_radius, cap=M)
        agents = spawn_cache[s]
        ox, oy = offs[w]
        for m, rec in enumerate(agents):
            valid[w, m] = True
            start_xy[w, m] = (rec.start[0] + ox, rec.start[1] + oy)
            goal_xy[w, m] = (rec.goal[0] + ox, rec.goal[1] + oy)
            start_yaw[w, m] = rec.start_heading
            state["x"][w, m] = rec.start[0] + ox
            state["y"][w, m] = rec.start[1] + oy
            state["yaw"][w, m] = rec.start_heading
            length[w, m] = rec.length
            width[w, m] = rec.width
        for m in range(len(agents), M):
            state["x"][w, m] = ox + OFFSTAGE_X
            state["y"][w, m] = oy
    r_hull, d_hull = circle_layout(length, width, params.wheelbase)
    tables, scene_of_world = scene_tables_of(worlds)
    return EngineTables(W, M, np.asarray(offs, dtype=np.float64), scene_of_world, tables, mu_eff,
                        weather, valid, start_xy, goal_xy, start_yaw, length, width,
                        r_hull, d_hull, state)


def compact_subset(worlds: WorldBatch, keep: np.ndarray) -> dict:
    """Dense (W, 1, K) lane/edge arrays in global coordinates, the shape the
    reference engine exposes as ``engine.lane`` / ``engine.edge``."""
    W = keep.shape[0]
    K = max(1, int(keep.sum(axis=1).max()))
    mid_g = worlds.midpoints + worlds.grid_offsets[:, None, :]
    out = {"mid": np.zeros((W, K, 2)), "dir": np.zeros((W, K, 2)), "half_len": np.zeros((W, K)),
           "half_wid": np.zeros((W, K)), "mask": np.zeros((W, K), dtype=bool)}
    for w in range(W):
        idx = np.nonzero(keep[w])[0]
        n = len(idx)
        out["mid"][w, :n] = mid_g[w, idx]
        out["dir"][w, :n] = worlds.directions[w, idx]
        out["half_len"][w, :n] = worlds.half_lengths[w, idx]
        out["half_wid"][w, :n] = worlds.half_widths[w, idx]
        out["mask"][w, :n] = True
    return {k: v[:, None] for k, v in out.items()}
