"""On-device world construction: the host side of
``dg_build_scenes`` / ``dg_build_worlds`` (csrc/dg_worlds.cu).

The reference builds a batch with O(W) Python loops -- ``build_world_batch``
(world.py:148-194) fills padded (W, P_max) arrays world by world, the Engine
constructor places every world's agents (engine.py:192-227) and compacts the
lane / edge subsets per world (engine.py:234-253), and ``eval.random_goals``
walks every agent's lane (config.py:236-278).  Here the host only flattens the
prepared scene pool (per scene, not per world), draws the Philox streams the
reference draws (the scene order of ``assign_scenes``, the goal distances) and
launches; every per-world table is written by the GPU straight into the
engine's device arrays.

* ``DeviceScenes``      -- per-scene segment tables, lane / edge lists, vertex
  arc lengths and the spawn filter, built on the device (one CTA per scene).
* ``DeviceWorldBatch``  -- drop-in for ``scenes.WorldBatch``: the engine builds
  from it on the device; the reference's padded arrays (``midpoints`` ...)
  and ``scenario_ids`` are produced only when read.  ``shard(lo, hi)`` is a
  rank's world range, built by that rank alone.
* ``engine_tables``     -- the spawn table / initial state on the device
  (``tables.EngineTables`` field names, CUDA tensors).

Bit-identical to the host build (tables.py / scenes.py / goals.py), which is
pinned to the reference (tests/golden/init_default.npz, goals_random.npz,
worlds_4096.npz); GPU tests: tests/test_gpu_worldgen.py.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .params import OFFSTAGE_X
from .scenes import GRID_PITCH, SEGMENT_GAP, SEGMENT_HALF_WIDTH, SegmentArray, assign_scenes


def _ptr(t):
    return None if t is None else ct.c_void_p(t.data_ptr())


def _stream(device):
    return ct.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def scene_order(num_scenes: int, mode: str, seed: int) -> np.ndarray:
    """World w takes scene order[w % S] (assign_scenes, world.py:131-145): the
    Philox permutation of the pool for random_fill, the identity for fixed."""
    return np.asarray(assign_scenes(num_scenes, num_scenes, mode, seed), dtype=np.int32)


def flatten_pool(scenes) -> dict:
    """The prepared pool as flat arrays (DgScenePool), one pass over the scenes."""
    pts, starts, types, scene_poly, agents, scene_agent = [], [0], [], [0], [], [0]
    for spec in scenes:
        for p in spec.polylines:
            xy = np.asarray(p.points, dtype=np.float64)[:, :2]
            if len(xy) == 0:
                raise ValueError(f"scene {spec.scenario_id!r}: empty polyline")
            pts.append(xy)
            starts.append(starts[-1] + len(xy))
            types.append(int(p.type_code))
        scene_poly.append(len(types))
        for a in spec.agents:
            agents.append((a.start[0], a.start[1], a.start_heading, a.goal[0], a.goal[1], a.length, a.width))
        scene_agent.append(len(agents))
    return {
        "points": np.ascontiguousarray(np.concatenate(pts) if pts else np.zeros((0, 2))),
        "poly_start": np.asarray(starts, dtype=np.int32),
        "poly_type": np.asarray(types, dtype=np.int32),
        "scene_poly": np.asarray(scene_poly, dtype=np.int32),
        "agents": np.asarray(agents, dtype=np.float64).reshape(-1, 7),
        "scene_agent": np.asarray(scene_agent, dtype=np.int32),
    }


@dataclass
class DeviceScenes:
    """dg_build_scenes output for a pool (device tensors + the per-scene counts
    on the host, read once)."""

    device: torch.device
    num_scenes: int
    cap: int
    pool: dict                     # DgScenePool arrays (device)
    seg: dict                      # DgSceneSegments arrays (device)
    base: np.ndarray               # (S,) first pair row of each scene
    counts: dict                   # seg / lane / edge / lane_polys / kept per scene (host)
    desc_pool: N.DgScenePool = field(repr=False, default=None)
    desc_seg: N.DgSceneSegments = field(repr=False, default=None)
    _tables: tuple | None = field(repr=False, default=None)

    def scene_tables(self) -> tuple:
        """Per-scene SegmentArray host copies (scene-local), the WorldBatch's
        ``scene_tables``; one D2H copy of the segment rows."""
        if self._tables is None:
            host = {k: self.seg[k].cpu().numpy() for k in ("mid", "dir", "type", "half_len", "half_wid")}
            out = []
            for s in range(self.num_scenes):
                a, n = int(self.base[s]), int(self.counts["seg"][s])
                out.append(SegmentArray(host["mid"][a:a + n].copy(), host["dir"][a:a + n].copy(),
                                        host["type"][a:a + n].copy(), host["half_len"][a:a + n].copy(),
                                        host["half_wid"][a:a + n].copy()))
            self._tables = tuple(out)
        return self._tables


def build_scenes(scenes, device, gap=SEGMENT_GAP, bbox_half=100.0, goal_radius=3.0, cap=16) -> DeviceScenes:
    """Segments, lane / edge lists, arc tables and the spawn filter of every
    scene of the pool, on ``device`` (dg_build_scenes)."""
    if not scenes:
        raise ValueError("empty scene list")
    lib = N.load_library()
    dev = torch.device(device)
    flat = flatten_pool(scenes)
    S = len(scenes)
    n_pts, n_poly = len(flat["points"]), len(flat["poly_type"])
    pairs = max(1, n_pts - n_poly)
    pool = {k: torch.as_tensor(v).to(dev) for k, v in flat.items()}
    if pool["agents"].numel() == 0:
        pool["agents"] = torch.zeros((1, 7), dtype=torch.float64, device=dev)
    f64, i32 = dict(dtype=torch.float64, device=dev), dict(dtype=torch.int32, device=dev)
    seg = {"mid": torch.zeros((pairs, 2), **f64), "dir": torch.zeros((pairs, 2), **f64),
           "type": torch.zeros(pairs, **i32), "half_len": torch.zeros(pairs, **f64),
           "half_wid": torch.zeros(pairs, **f64), "lane_index": torch.zeros(pairs, **i32),
           "edge_index": torch.zeros(pairs, **i32), "arc": torch.zeros(max(1, n_pts), **f64),
           "seg_count": torch.zeros(S, **i32), "lane_count": torch.zeros(S, **i32),
           "edge_count": torch.zeros(S, **i32), "lane_polys": torch.zeros(S, **i32),
           "kept_count": torch.zeros(S, **i32), "kept_agent": torch.zeros(max(1, len(flat["agents"])), **i32)}
    dp = N.DgScenePool(num_scenes=S, num_polylines=n_poly, num_points=n_pts, num_agents=len(flat["agents"]),
                       **{k: pool[k].data_ptr() for k in ("points", "poly_start", "poly_type", "scene_poly",
                                                          "agents", "scene_agent")})
    db = N.DgSceneBuild(gap=float(gap), bbox_half=float(bbox_half), half_width=SEGMENT_HALF_WIDTH,
                        goal_radius=float(goal_radius), cap=int(cap))
    ds = N.DgSceneSegments(**{k: seg[k].data_ptr() for k in N.SCENE_SEG_FIELDS})
    N.check(lib, lib.dg_build_scenes(ct.byref(dp), ct.byref(db), ct.byref(ds), _stream(dev)), "dg_build_scenes")
    counts = torch.stack([seg[k] for k in ("seg_count", "lane_count", "edge_count", "lane_polys",
                                           "kept_count")]).cpu().numpy()
    base = flat["poly_start"][flat["scene_poly"][:-1]] - flat["scene_poly"][:-1]
    return DeviceScenes(dev, S, int(cap), pool, seg, base.astype(np.int64),
                        dict(zip(("seg", "lane", "edge", "lane_polys", "kept"), counts)), dp, ds)


class DeviceWorldBatch:
    """A world batch whose per-world tables are built on the GPU -- the drop-in
    for ``scenes.WorldBatch`` / ``drivegrid.world.WorldBatch`` (world.py:37-56).

    World w is world ``world_base + w`` of a batch of ``total_worlds``; the
    reference's padded arrays and per-world ids materialise only when read."""

    def __init__(self, scenes: DeviceScenes, scenario_ids: list, order: np.ndarray, num_worlds: int,
                 world_base: int = 0, total_worlds: int | None = None, pitch: float = GRID_PITCH):
        self.scenes = scenes
        self._ids = list(scenario_ids)
        self.order = np.asarray(order, dtype=np.int32)
        self.W = int(num_worlds)
        self.world_base = int(world_base)
        self.total_worlds = int(total_worlds if total_worlds is not None else num_worlds)
        self.pitch = float(pitch)
        self.grid_cols = int(np.ceil(np.sqrt(self.total_worlds)))
        self._order_dev = torch.as_tensor(self.order).to(scenes.device)
        self._padded = None
        self._world = None

    # -- WorldBatch surface
    @property
    def num_worlds(self) -> int:
        return self.W

    @property
    def scene_index(self) -> np.ndarray:
        g = self.world_base + np.arange(self.W)
        return self.order[g % len(self.order)].astype(np.int64)

    @property
    def scene_tables(self) -> tuple:
        return self.scenes.scene_tables()

    @property
    def p_max(self) -> int:
        used = np.unique(self.order if self.W >= len(self.order) else self.scene_index)
        return max(1, int(self.scenes.counts["seg"][used].max()))

    @property
    def scenario_ids(self) -> list:
        return [self._ids[s] for s in self.scene_index]

    @property
    def grid_offsets(self) -> np.ndarray:
        return self._world_arrays()["grid_offset"].cpu().numpy()

    def _padded_arrays(self) -> dict:
        if self._padded is None:
            self._padded = {k: v.cpu().numpy() for k, v in self.build(padded=True)["padded"].items()}
        return self._padded

    midpoints = property(lambda self: self._padded_arrays()["wb_mid"])
    directions = property(lambda self: self._padded_arrays()["wb_dir"])
    type_codes = property(lambda self: self._padded_arrays()["wb_type"])
    half_lengths = property(lambda self: self._padded_arrays()["wb_half_len"])
    half_widths = property(lambda self: self._padded_arrays()["wb_half_wid"])
    mask = property(lambda self: self._padded_arrays()["wb_mask"].astype(bool))

    def shard(self, lo: int, hi: int) -> "DeviceWorldBatch":
        """Worlds [lo, hi) of this batch (a rank's share; built by that rank)."""
        return DeviceWorldBatch(self.scenes, self._ids, self.order, hi - lo, self.world_base + lo,
                                self.total_worlds, self.pitch)

    # -- device builds
    def _world_arrays(self) -> dict:
        if self._world is None:
            self._world = self.build()["world"]
        return self._world

    def build(self, M: int | None = None, wheelbase: float = 2.6, spawn: dict | None = None,
              padded: bool = False, subsets: tuple = (), goals: dict | None = None) -> dict:
        """One dg_build_worlds launch sequence.  ``spawn``: the engine's device
        arrays to fill (valid, alive, start_xy, goal_xy, start_yaw, length,
        width, r_hull, d_hull, state); ``goals``: {min, max, draws (device f64)}
        (needs spawn's start_xy / goal_xy, or with ``spawn`` None the
        ``goal_xy`` / ``start_xy`` entries of ``goals``); ``subsets``: any of
        "lane", "edge" (_compact_subset, [W][K]); ``padded``: the WorldBatch
        arrays [W][p_max]."""
        lib = N.load_library()
        sc = self.scenes
        dev = sc.device
        W = self.W
        M = int(M if M is not None else sc.cap)
        if M != sc.cap:
            raise ValueError(f"scenes were filtered for {sc.cap} agents per world, not {M}")
        f64, i32, u8 = (dict(dtype=d, device=dev) for d in (torch.float64, torch.int32, torch.uint8))
        world = {"assignment": torch.empty(W, **i32), "grid_offset": torch.empty((W, 2), **f64)}
        b = N.DgWorldBuild(W=W, M=M, num_scenes=sc.num_scenes, grid_cols=self.grid_cols,
                           world_base=self.world_base, pitch=self.pitch, offstage_x=OFFSTAGE_X,
                           wheelbase=float(wheelbase), scene_order=self._order_dev.data_ptr())
        b.assignment, b.grid_offset = world["assignment"].data_ptr(), world["grid_offset"].data_ptr()
        if spawn is not None:
            for k in N.WORLD_OUT_FIELDS[2:]:
                if spawn.get(k) is not None:
                    setattr(b, k, spawn[k].data_ptr())
        out = {"world": world}
        keep = []
        if goals is not None:
            b.random_goals, b.goal_min, b.goal_max = 1, float(goals["min"]), float(goals["max"])
            if goals.get("draws") is not None:
                b.goal_draws = goals["draws"].data_ptr()
            if spawn is None:
                b.start_xy, b.goal_xy = goals["start_xy"].data_ptr(), goals["goal_xy"].data_ptr()
        if padded:
            P = self.p_max
            pad = {"wb_mid": torch.empty((W, P, 2), **f64), "wb_dir": torch.empty((W, P, 2), **f64),
                   "wb_type": torch.empty((W, P), **i32), "wb_half_len": torch.empty((W, P), **f64),
                   "wb_half_wid": torch.empty((W, P), **f64), "wb_mask": torch.empty((W, P), **u8)}
            b.p_max = P
            for k, v in pad.items():
                setattr(b, k, v.data_ptr())
            out["padded"] = pad
        for sub in subsets:
            K = max(1, int(sc.counts[sub][np.unique(self.scene_index)].max()))
            arr = {"mid": torch.empty((W, K, 2), **f64), "dir": torch.empty((W, K, 2), **f64),
                   "half_len": torch.empty((W, K), **f64), "half_wid": torch.empty((W, K), **f64),
                   "mask": torch.empty((W, K), **u8)}
            setattr(b, f"k_{sub}", K)
            for k, v in arr.items():
                setattr(b, f"{sub}_{k}", v.data_ptr())
            out[sub] = arr
        keep.append(b)
        N.check(lib, lib.dg_build_worlds(ct.byref(sc.desc_pool), ct.byref(sc.desc_seg), ct.byref(b), _stream(dev)),
                "dg_build_worlds")
        return out

    def compact_subset(self, sub: str) -> dict:
        """Engine.lane / Engine.edge (engine.py:234-253) as host arrays (W, 1, K)."""
        arr = self.build(subsets=(sub,))[sub]
        host = {k: v.cpu().numpy() for k, v in arr.items()}
        host["mask"] = host["mask"].astype(bool)
        return {k: v[:, None] for k, v in host.items()}

    def goal_draw_count(self) -> int:
        """Draws of Philox stream (seed, 4) that worlds [0, world_base + W) consume."""
        c = self.scenes.counts
        per_scene = np.where(c["lane_polys"] > 0, c["kept"], 0).astype(np.int64)
        g = np.arange(self.world_base + self.W)
        return int(per_scene[self.order[g % len(self.order)]].sum())


def build_world_batch(scenes, num_worlds: int, device, mode: str = "random_fill", seed: int = 42,
                      gap: float = SEGMENT_GAP, bbox_half: float = 100.0, goal_radius: float = 3.0,
                      cap: int = 16):
    """``scenes.build_world_batch`` with the per-world work on the GPU:
    (DeviceWorldBatch, assignment)."""
    dsc = build_scenes(scenes, device, gap=gap, bbox_half=bbox_half, goal_radius=goal_radius, cap=cap)
    order = scene_order(len(scenes), mode, seed)
    batch = DeviceWorldBatch(dsc, [s.scenario_id for s in scenes], order, num_worlds)
    return batch, batch.scene_index


@dataclass
class DeviceEngineTables:
    """``tables.EngineTables`` with the per-(world, agent) arrays on the device
    (the spawn table and initial state written by dg_build_worlds) and host
    copies of the ones the Engine exposes as numpy attributes."""

    W: int
    M: int
    grid_offsets: np.ndarray
    scene_of_world: np.ndarray
    scenes: list
    mu_eff: np.ndarray
    weather: np.ndarray
    dev: dict
    valid: np.ndarray
    length: np.ndarray
    width: np.ndarray
    r_hull: np.ndarray
    d_hull: np.ndarray


def engine_tables(worlds: DeviceWorldBatch, frictions, config, params) -> DeviceEngineTables:
    from .tables import _scene_table, world_friction

    W, M = config.num_envs, config.num_agents
    if worlds.num_worlds != W:
        raise ValueError(f"world batch has {worlds.num_worlds} worlds, config wants {W}")
    if len(frictions) != W:
        raise ValueError("need one friction assignment per world")
    mu_eff, weather = world_friction(frictions, params)
    dev = worlds.scenes.device
    f64 = dict(dtype=torch.float64, device=dev)
    d = {"valid": torch.empty((W, M), dtype=torch.uint8, device=dev),
         "alive": torch.empty((W, M), dtype=torch.uint8, device=dev),
         "start_xy": torch.empty((W, M, 2), **f64), "goal_xy": torch.empty((W, M, 2), **f64),
         "start_yaw": torch.empty((W, M), **f64), "length": torch.empty((W, M), **f64),
         "width": torch.empty((W, M), **f64), "r_hull": torch.empty((W, M), **f64),
         "d_hull": torch.empty((W, M), **f64), "state": torch.empty((12, W, M), **f64)}
    out = worlds.build(M=M, wheelbase=params.wheelbase, spawn=d)
    d["assignment"], d["grid_offset"] = out["world"]["assignment"], out["world"]["grid_offset"]
    host = {k: d[k].cpu().numpy() for k in ("valid", "length", "width", "r_hull", "d_hull", "grid_offset")}
    return DeviceEngineTables(W, M, host["grid_offset"], worlds.scene_index,
                              [_scene_table(s) for s in worlds.scene_tables], mu_eff, weather, d,
                              host["valid"].astype(bool), host["length"], host["width"], host["r_hull"],
                              host["d_hull"])


def resample_goals(engine, cfg) -> None:
    """eval.random_goals on the device (config.py:236-278): the engine's goals
    are rewritten in place from its start positions; distances from Philox
    stream (seed, 4) exactly as the reference draws them."""
    worlds = engine.worlds
    lo, hi = float(cfg.eval.goal_min_m), float(cfg.eval.goal_max_m)
    draws = None
    if lo != hi:
        n = worlds.goal_draw_count()
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([cfg.seed, 4])))
        # rng.uniform(lo, hi) once per valid agent == one vector draw of the same length
        draws = torch.as_tensor(rng.uniform(lo, hi, size=max(n, 1))).to(engine.device)
    d = engine.device_tables()
    worlds.build(M=engine.M, goals={"min": lo, "max": hi, "draws": draws, "start_xy": d["start_xy"],
                                    "goal_xy": d["goal_xy"]})
