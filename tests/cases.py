"""Seeded parity cases shared by the CPU (oracle vs golden) and GPU (kernel vs
oracle) tests.  Each case mirrors one generator in ``tests/golden/make_golden.py``
but is built from this repo's own host-init layer, so it runs on the GPU box
where the reference tree does not exist.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.friction import SURFACE_ORDER, assign_friction
from paper_2605_08528_b200.params import ObsConfig, SimConfig
from paper_2605_08528_b200.policies import LaneFollower
from paper_2605_08528_b200.scenes import (build_world_batch, export_world_batch, import_world_batch, prepare_scene,
                                          straight_scene)

GOLDEN = Path(__file__).resolve().parent / "golden"


def cfg_of(W, M, seed=42, mode="dynamic", assignment="random_fill", invincible=False,
           episode_len=1500):
    cfg = C.RootConfig()
    cfg.env.num_envs = W
    cfg.env.num_agents_per_env = M
    cfg.env.dynamics_mode = mode
    cfg.env.episode_len = episode_len
    cfg.eval.invincible = invincible
    cfg.seed = seed
    cfg.scene_factory.assignment_mode = assignment
    return cfg


def philox_actions(seed, T, W, M):
    g = np.random.Generator(np.random.Philox(seed))
    return g.uniform(-1.0, 1.0, (T, W, M, 3)).astype(np.float32)


def event_actions(T, W, M):
    steer = np.array([0.0, 0.08, -0.08, 0.3, -0.3, 0.02, -0.5, 0.15, 0.0, -0.15, 1.0,
                      -0.02, 0.6, 0.0, -1.0, 0.04])[:M]
    acts = np.zeros((T, W, M, 3), dtype=np.float32)
    acts[..., 0] = 1.0
    acts[..., 1] = steer[None, None, :] * (1.0 - 0.25 * (np.arange(W)[None, :, None] % 2))
    rows = (np.arange(M) % 5 == 0)
    acts[100:160, :, rows, 2] = 1.0
    acts[100:160, :, rows, 0] = -1.0
    return acts


def wet_frictions(W):
    films = (0.0, 0.3, 0.5, 0.8, 1.0, 2.0)
    return [assign_friction(SURFACE_ORDER[(w // len(films)) % 3], films[w % len(films)])
            for w in range(W)]


@dataclass
class Case:
    name: str
    inputs: C.EngineInputs
    actions: np.ndarray | None = None     # (T, W, M, 3) float32, None = LaneFollower
    steps: int = 0
    full_obs_steps: tuple = field(default_factory=tuple)


def case_inputs(name: str) -> Case:
    if name == "traj_c1":
        scene = prepare_scene(straight_scene(agent_count=1, goal_dist=50.0))
        inp = C.build_inputs(cfg_of(1, 1, invincible=True, episode_len=2000), scenes=[scene])
        return Case(name, inp, philox_actions(3, 1000, 1, 1), 1000, tuple(range(1, 1001)))
    if name == "traj_pool":
        return Case(name, C.build_inputs(cfg_of(4, 16)), None, 60, (1, 24, 25, 60))
    if name == "traj_wet":
        W, M = 12, 16
        cfg = cfg_of(W, M, seed=5)
        inp = C.build_inputs(cfg)
        pool = inp.scenes
        worlds, assignment = build_world_batch(pool, W, mode="random_fill", seed=5)
        inp.worlds, inp.assignment, inp.frictions = worlds, assignment, wet_frictions(W)
        inp.sim = SimConfig(num_envs=W, num_agents=M, seed=5)
        acts = philox_actions(9, 80, W, M)
        acts[..., 0] = np.abs(acts[..., 0])
        return Case(name, inp, acts, 80, (1, 40, 80))
    if name == "traj_bicycle":
        inp = C.build_inputs(cfg_of(2, 3, mode="bicycle", assignment="fixed", seed=11))
        return Case(name, inp, philox_actions(4, 50, 2, 3), 50, (1, 50))
    if name == "traj_custom_obs":
        cfg = cfg_of(2, 5, assignment="fixed", seed=19)
        cfg.obs = ObsConfig(include_weather=False, k_road=20, k_vehicles=3, road_radius=12.5)
        return Case(name, C.build_inputs(cfg), philox_actions(6, 40, 2, 5), 40, tuple(range(1, 41)))
    if name == "traj_timeout":
        return Case(name, C.build_inputs(cfg_of(2, 16, seed=17, episode_len=25)), None, 40, (1, 25, 26, 40))
    if name == "traj_sparse":
        scene = prepare_scene(straight_scene(agent_count=2, goal_dist=40.0))
        inp = C.build_inputs(cfg_of(3, 4, seed=13), scenes=[scene])
        return Case(name, inp, philox_actions(12, 60, 3, 4), 60, (1, 30, 60))
    if name in ("traj_obs_min", "traj_obs_one"):
        cfg = cfg_of(3, 6, seed=29)
        kr = kv = 0 if name == "traj_obs_min" else 1
        cfg.obs = ObsConfig(include_weather=name == "traj_obs_min", k_road=kr, k_vehicles=kv)
        return Case(name, C.build_inputs(cfg), philox_actions(14, 40, 3, 6), 40, (1, 20, 40))
    if name == "traj_no_edges":
        from paper_2605_08528_b200.scenes import AgentRecord, Polyline, ScenarioSpec
        xs = np.arange(-80.0, 80.01, 2.0)

        def row(y):
            return np.stack([xs, np.full_like(xs, y), np.zeros_like(xs)], axis=1)

        agents = [AgentRecord(f"a{i}", (-70.0 + 15.0 * i, 3.5 * (i % 2)), 0.0, (-20.0 + 15.0 * i, 3.5 * (i % 2)))
                  for i in range(4)]
        spec = ScenarioSpec("no_edges", [Polyline(1, row(0.0)), Polyline(2, row(3.5)), Polyline(6, row(7.0))], agents)
        return Case(name, C.build_inputs(cfg_of(2, 4, seed=41), scenes=[prepare_scene(spec)]), None, 50, (1, 50))
    if name == "traj_dense":
        lanes = tuple(float(x) for x in np.round(np.arange(-9.0, 9.01, 0.25), 2))
        scene = prepare_scene(straight_scene("dense", lane_offsets=lanes, agent_count=8, agent_gap=15.0,
                                             goal_dist=40.0))
        return Case(name, C.build_inputs(cfg_of(2, 8, seed=3), scenes=[scene]), None, 30, (1, 30))
    if name == "traj_forge":
        inp = C.build_inputs(cfg_of(6, 16, seed=23))
        inp.worlds = forge_roundtrip(inp.worlds)[1]
        inp.sim = SimConfig(num_envs=6, num_agents=16, seed=23)
        return Case(name, inp, None, 40, (1, 40))
    if name in ("traj_events", "traj_events_inv"):
        inp = C.build_inputs(cfg_of(4, 16, seed=31, invincible=name.endswith("_inv")))
        return Case(name, inp, event_actions(420, 4, 16), 420, (1, 150, 420))
    raise KeyError(name)


TRAJ_CASES = ("traj_c1", "traj_pool", "traj_wet", "traj_bicycle", "traj_custom_obs",
              "traj_events", "traj_events_inv", "traj_sparse", "traj_timeout", "traj_forge",
              "traj_dense", "traj_obs_min", "traj_obs_one", "traj_no_edges")


def forge_roundtrip(worlds):
    """(bytes of the binary world export, the batch imported back from them)."""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "worlds.bin"
        export_world_batch(worlds, path)
        return path.read_bytes(), import_world_batch(path)


def run_case(engine, case: Case, on_step):
    """Drive ``engine`` (oracle or GPU) through the case; ``on_step(t, out,
    actions)`` sees every step (t is 1-based)."""
    if case.actions is None:
        pol = LaneFollower(obs_config=engine.obs_config)
        obs = np.asarray(engine.observe())
        for t in range(case.steps):
            a = pol(obs)
            out = engine.step(a)
            on_step(t + 1, out, a)
            obs = np.asarray(out.obs)
    else:
        for t in range(case.steps):
            a = case.actions[t].astype(np.float64)
            out = engine.step(a)
            on_step(t + 1, out, a)


# ---------------------------------------------------------------- world construction
def worlds_case_pool():
    """The prepared scene_cases pool (make_golden.worlds_cases)."""
    import types

    import sys

    from paper_2605_08528_b200 import scenes as S
    if str(GOLDEN) not in sys.path:
        sys.path.insert(0, str(GOLDEN))
    from scene_cases import scene_specs
    mod = types.SimpleNamespace(Polyline=S.Polyline, AgentRecord=S.AgentRecord, ScenarioSpec=S.ScenarioSpec,
                                straight_scene=S.straight_scene, crossroads_scene=S.crossroads_scene,
                                two_level_scene=S.two_level_scene, shift_scenario=S.shift_scenario)
    return [p for p in map(prepare_scene, scene_specs(mod)) if p is not None]


def world_cfg(W, M=16, seed=42, goals=None):
    cfg = cfg_of(W, M, seed=seed)
    if goals is not None:
        cfg.eval.random_goals, cfg.eval.goal_min_m, cfg.eval.goal_max_m = True, goals[0], goals[1]
    return cfg


def canon(a):
    a = np.asarray(a)
    if a.dtype.kind == "f":
        a = a.astype(np.float64)
    elif a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return np.ascontiguousarray(a)


def host_world_arrays(cfg, scenes=None) -> dict:
    """The init tables of the host build (scenes / tables / goals restatement),
    keyed like make_golden._world_arrays."""
    from paper_2605_08528_b200.goals import resample_goals
    from paper_2605_08528_b200.params import STATE_FIELDS
    from paper_2605_08528_b200.tables import build_tables, compact_subset, edge_mask_of, lane_mask_of
    inp = C.build_inputs(cfg, scenes)
    w = inp.worlds
    t = build_tables(w, inp.scenes, inp.assignment, inp.frictions, inp.sim, inp.params)
    goal_xy = t.goal_xy
    if cfg.eval.random_goals:
        goal_xy = resample_goals(t.goal_xy, t.start_xy, t.valid, w.grid_offsets, inp.scenes, inp.assignment, cfg)
    out = {"midpoints": w.midpoints, "directions": w.directions, "type_codes": w.type_codes,
           "half_lengths": w.half_lengths, "half_widths": w.half_widths, "mask": w.mask,
           "grid_offsets": w.grid_offsets, "valid": t.valid, "start_xy": t.start_xy, "goal_xy": goal_xy,
           "start_yaw": t.start_yaw, "length": t.length, "width": t.width, "r_hull": t.r_hull,
           "d_hull": t.d_hull, "scenario_ids": np.frombuffer("\n".join(w.scenario_ids).encode(), np.uint8)}
    for sub, fn in (("lane", lane_mask_of), ("edge", edge_mask_of)):
        for k, v in compact_subset(w, fn(w.type_codes, w.mask)).items():
            out[f"{sub}_{k}"] = v
    for k in STATE_FIELDS:
        out["state_" + k] = t.state0[k]
    return out


def engine_world_arrays(eng) -> dict:
    """The same tables read back from a GPU engine (device world construction)."""
    from paper_2605_08528_b200.params import STATE_FIELDS
    w = eng.worlds
    out = {"midpoints": w.midpoints, "directions": w.directions, "type_codes": w.type_codes,
           "half_lengths": w.half_lengths, "half_widths": w.half_widths, "mask": w.mask,
           "grid_offsets": w.grid_offsets, "valid": eng.valid, "start_xy": eng.start_xy,
           "goal_xy": eng.goal_xy, "start_yaw": eng.start_yaw, "length": eng.length, "width": eng.width,
           "r_hull": eng.r_hull, "d_hull": eng.d_hull,
           "scenario_ids": np.frombuffer("\n".join(w.scenario_ids).encode(), np.uint8)}
    for sub in ("lane", "edge"):
        for k, v in getattr(eng, sub).items():
            out[f"{sub}_{k}"] = v
    st = eng.state
    for k in STATE_FIELDS:
        out["state_" + k] = st[k]
    return out


def check_world_hashes(arrays: dict, golden, tag: str) -> None:
    import hashlib
    for k, v in arrays.items():
        c = canon(v)
        want = bytes(golden[f"{tag}__{k}__sha"]).decode()
        assert tuple(c.shape) == tuple(golden[f"{tag}__{k}__shape"]), (tag, k, c.shape)
        assert hashlib.sha256(c.tobytes()).hexdigest() == want, f"{tag}: {k} differs from the reference"
