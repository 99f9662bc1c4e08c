"""Generate the golden fixtures from the reference package (run in the dev container).

The reference (``/root/reference/pkg``) is pure Python + numpy; it is imported
read-only from its source tree and never travels to the GPU box.  This script
records what the reference computes for a set of seeded cases; the CPU tests
pin the oracle restatement (``oracle/``) and the host-init layer of the product
against these files.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Cases (each an .npz under tests/golden/):
  init_default      256x16 default pool: world tables, spawn table, mu, weather
  friction          mu_effective / assign_friction over surfaces x film depths
  traj_c1           1x1 straight road, invincible, 1000 fp32 Philox(3) actions
  traj_pool         4x16 default pool (random_fill, seed 42), LaneFollower, 60 steps
  traj_wet          12x16 default pool, per-world friction sweep, fp32 random actions
  traj_bicycle      2x3 bicycle backend, random actions
  traj_custom_obs   2x5, reduced ObsConfig (no weather, k_road 20, k_vehicles 3)
  traj_reset        2x4: steps, EnvHandle.reset quirk, overlapping teleport starts
  traj_events       4x16, scripted throttle/steer/brake: goal, edge, crash, collision
  traj_events_inv   same actions, invincible mode (latched events, no termination)
  drac_wet          traj_wet's run through Engine.run_episode(record=True): per-step
                    pairwise_drac + episode_metrics (metrics.py:33-125)
  drac_events       traj_events' run, same records (collisions, DRAC > 3.4)
  traj_timeout      2x16 default pool, episode_len 25, 40 LaneFollower steps: every
                    survivor times out (reason 5, not parked), then steps dead
  traj_sparse       3x4 on a 2-agent straight road: half the slots invalid (never alive,
                    masked everywhere), random actions
  worlds_4096       sha256 of every init table of build_engine at 4096x16 (plain and
                    eval.random_goals) -- the on-device world construction pins
  worlds_cases      the scene_cases pool at 29 worlds: full init tables (+ random goals)
  sysid             sysid.py: maneuver sets, 60 Hz channel rollouts of 6 candidate
                    parameter vectors on one maneuver of every kind, sysid_loss,
                    and a small five-stage run_cem (population 8, 40 trials)
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("DRIVEGRID_REF", "/root/reference/pkg"))
sys.dont_write_bytecode = True
sys.path[:0] = [str(REF / "src"), str(REF / "bindings" / "src")]
sys.path.insert(0, str(Path(__file__).resolve().parent))

from drivegrid import vehicle as vh  # noqa: E402
from drivegrid.config import RootConfig, build_engine, prepare_scene  # noqa: E402
from drivegrid.friction import SURFACE_ORDER, assign_friction, mu_effective  # noqa: E402
from drivegrid.observation import ObsConfig  # noqa: E402
from drivegrid.policies import LaneFollower  # noqa: E402
from drivegrid.synth import default_scene_pool, straight_scene  # noqa: E402

OUT = Path(__file__).resolve().parent
EVENTS = ("goal", "collision", "crash", "lane_forbidden")
TERMS = ("progress", "lane", "offroad", "idle", "ttc_vehicle", "ttc_edge", "total")


def cfg_of(W, M, seed=42, mode="dynamic", assignment="random_fill", invincible=False,
           episode_len=1500):
    cfg = RootConfig()
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


class Recorder:
    """Per-step outputs; full obs only at the listed steps (1-based)."""

    def __init__(self, full_obs_steps=()):
        self.full_steps = set(full_obs_steps)
        self.rows = {}
        self.obs_full = {}

    def add(self, t, eng, out, actions):
        row = {
            "actions": np.asarray(actions, dtype=np.float64),
            "rewards": out.rewards, "dones": out.dones,
            "reason": out.info["reason"], "alive": out.info["alive"],
            "alive_pre": out.info["alive_pre"], "ttc_min": out.info["ttc_min"],
            "obs_sum": out.obs.astype(np.float64).sum(axis=-1),
            "obs_abs": np.abs(out.obs.astype(np.float64)).sum(axis=-1),
            "obs_nnz": (out.obs != 0).sum(axis=-1),
            "obs_ego": out.obs[..., :16].copy(),
        }
        for k in EVENTS:
            row["ev_" + k] = out.events[k]
        for k in TERMS:
            row["term_" + k] = out.info["reward_terms"][k]
        for k in vh.STATE_FIELDS:
            row["snap_" + k] = out.info["state"][k]
            row["state_" + k] = eng.state[k]
        for k, v in row.items():
            self.rows.setdefault(k, []).append(np.asarray(v))
        if t in self.full_steps:
            self.obs_full[t] = out.obs.copy()

    def save(self, name, **extra):
        arrays = {k: np.stack(v) for k, v in self.rows.items()}
        for t, o in self.obs_full.items():
            arrays[f"obs_full_{t}"] = o
        arrays.update(extra)
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        print(name, sum(a.nbytes for a in arrays.values()) // 1024, "KiB raw")


def run_actions(eng, actions, rec):
    for t in range(actions.shape[0]):
        out = eng.step(actions[t].astype(np.float64))
        rec.add(t + 1, eng, out, actions[t])


def init_default():
    eng = build_engine(cfg_of(256, 16))
    w = eng.worlds
    np.savez_compressed(
        OUT / "init_default.npz",
        midpoints=w.midpoints, directions=w.directions, type_codes=w.type_codes,
        half_lengths=w.half_lengths, half_widths=w.half_widths, mask=w.mask,
        grid_offsets=w.grid_offsets, mu_eff=eng.mu_eff, weather=eng.weather,
        valid=eng.valid, start_xy=eng.start_xy, goal_xy=eng.goal_xy, length=eng.length,
        width=eng.width, r_hull=eng.r_hull, d_hull=eng.d_hull,
        lane_mid=eng.lane["mid"], edge_mid=eng.edge["mid"],
        **{"state_" + k: eng.state[k] for k in vh.STATE_FIELDS},
        obs0=eng.observe())
    print("init_default")


def friction():
    films = np.array([0.0, 0.1, 0.3, 0.5, 0.8, 0.86, 1.0, 2.0])
    mu_s = np.array([[mu_effective(s, h) for h in films] for s in SURFACE_ORDER])
    mu_d = np.array([[mu_effective(s, h, slip=0.8) for h in films] for s in SURFACE_ORDER])
    asg = np.array([[assign_friction(s, h).mu_static for h in films] for s in SURFACE_ORDER])
    np.savez_compressed(OUT / "friction.npz", films=films, mu_static=mu_s, mu_dynamic=mu_d,
                        assigned=asg)
    print("friction")


def friction_table():
    """mu_effective of the reference over a dense film sweep (the vectorised
    host table, friction.mu_table, must reproduce it)."""
    g = np.random.Generator(np.random.Philox(21))
    films = np.concatenate([[0.0, 1e-9, 0.3, 0.86, 1.0, 2.0, 5.0], g.uniform(0.0, 3.0, 993)])
    slips = np.array([0.15, 0.8, 0.5, 1.0, 0.0])
    mu = np.array([[[mu_effective(s, float(h), slip=float(sl)) for h in films] for sl in slips]
                   for s in SURFACE_ORDER])
    np.savez_compressed(OUT / "friction_table.npz", films=films, slips=slips, mu=mu)
    print("friction_table")


def traj_c1():
    scene = prepare_scene(straight_scene(agent_count=1, goal_dist=50.0))
    eng = build_engine(cfg_of(1, 1, invincible=True, episode_len=2000), scenes=[scene])
    rec = Recorder(full_obs_steps=range(1, 1001))
    run_actions(eng, philox_actions(3, 1000, 1, 1), rec)
    rec.save("traj_c1")


def traj_pool():
    eng = build_engine(cfg_of(4, 16))
    pol = LaneFollower(obs_config=eng.obs_config)
    rec = Recorder(full_obs_steps=(1, 24, 25, 60))
    obs = eng.observe()
    obs0 = obs.copy()
    for t in range(60):
        a = pol(obs)
        out = eng.step(a)
        rec.add(t + 1, eng, out, a)
        obs = out.obs
    rec.save("traj_pool", obs0=obs0)


def wet_frictions(W):
    films = (0.0, 0.3, 0.5, 0.8, 1.0, 2.0)
    out = []
    for w in range(W):
        s = SURFACE_ORDER[(w // len(films)) % 3]
        out.append(assign_friction(s, films[w % len(films)]))
    return out


def traj_wet():
    from drivegrid.config import load_scene_pool
    from drivegrid.engine import Engine, SimConfig
    from drivegrid.world import build_world_batch

    W, M = 12, 16
    cfg = cfg_of(W, M, seed=5)
    pool = load_scene_pool(cfg.scene_factory)
    worlds, assignment = build_world_batch(pool, W, mode="random_fill", seed=5)
    fr = wet_frictions(W)
    eng = Engine(worlds, pool, assignment, fr, SimConfig(num_envs=W, num_agents=M, seed=5))
    rec = Recorder(full_obs_steps=(1, 40, 80))
    acts = philox_actions(9, 80, W, M)
    acts[..., 0] = np.abs(acts[..., 0])  # keep agents moving so crash/edge events occur
    run_actions(eng, acts, rec)
    rec.save("traj_wet", mu_eff=eng.mu_eff, weather=eng.weather,
             films=np.array([f.water_film_mm for f in fr]),
             surfaces=np.array([SURFACE_ORDER.index(f.surface.name) for f in fr]))


def traj_bicycle():
    eng = build_engine(cfg_of(2, 3, mode="bicycle", assignment="fixed", seed=11))
    rec = Recorder(full_obs_steps=(1, 50))
    run_actions(eng, philox_actions(4, 50, 2, 3), rec)
    rec.save("traj_bicycle")


def traj_obs_min():
    """Degenerate observation sizes: no road rows and no neighbour rows
    (ego block only), with weather; then one road row and one neighbour row."""
    for name, kr, kv, weather in (("traj_obs_min", 0, 0, True), ("traj_obs_one", 1, 1, False)):
        cfg = cfg_of(3, 6, seed=29)
        cfg.obs = ObsConfig(include_weather=weather, k_road=kr, k_vehicles=kv)
        eng = build_engine(cfg)
        rec = Recorder(full_obs_steps=(1, 20, 40))
        run_actions(eng, philox_actions(14, 40, 3, 6), rec)
        rec.save(name)


def no_edge_scene(Polyline, AgentRecord, ScenarioSpec):
    """Lane centres of both lane codes and an unrelated polyline, no road edge
    at all (the edge subset is empty)."""
    xs = np.arange(-80.0, 80.01, 2.0)

    def row(y, z=0.0):
        return np.stack([xs, np.full_like(xs, y), np.full_like(xs, z)], axis=1)

    agents = [AgentRecord(f"a{i}", (-70.0 + 15.0 * i, 3.5 * (i % 2)), 0.0, (-20.0 + 15.0 * i, 3.5 * (i % 2)))
              for i in range(4)]
    return ScenarioSpec("no_edges", [Polyline(1, row(0.0)), Polyline(2, row(3.5)), Polyline(6, row(7.0))], agents)


def traj_no_edges():
    from drivegrid.scenario import AgentRecord, Polyline, ScenarioSpec
    scene = prepare_scene(no_edge_scene(Polyline, AgentRecord, ScenarioSpec))
    eng = build_engine(cfg_of(2, 4, seed=41), scenes=[scene])
    pol = LaneFollower(obs_config=eng.obs_config)
    rec = Recorder(full_obs_steps=(1, 50))
    obs = eng.observe()
    for t in range(50):
        a = pol(obs)
        out = eng.step(a)
        rec.add(t + 1, eng, out, a)
        obs = out.obs
    rec.save("traj_no_edges")


def scene_verdicts():
    """reject_degenerate_scene / prepare_scene / filter_agents over the
    synthetic specs of scene_cases.py (scenario.py:169-260, config.py:162-168)."""
    import json
    import types

    from drivegrid import scenario as sc
    from drivegrid import synth
    from scene_cases import scene_specs
    mod = types.SimpleNamespace(Polyline=sc.Polyline, AgentRecord=sc.AgentRecord, ScenarioSpec=sc.ScenarioSpec,
                                straight_scene=synth.straight_scene, crossroads_scene=synth.crossroads_scene,
                                two_level_scene=synth.two_level_scene, shift_scenario=sc.shift_scenario)
    out, arrays = [], {}
    for i, spec in enumerate(scene_specs(mod)):
        v = sc.reject_degenerate_scene(spec)
        rec = {"id": spec.scenario_id, "accepted": bool(v.accepted), "reason": v.reason}
        p = prepare_scene(spec)
        if p is not None:
            kept = sc.filter_agents(p)
            rec["kept"] = len(kept)
            arrays[f"s{i}_points"] = np.concatenate([q.points for q in p.polylines])
            arrays[f"s{i}_agents"] = np.array([[*a.start, a.start_heading, *a.goal, a.length, a.width]
                                                for a in p.agents])
        out.append(rec)
    np.savez_compressed(OUT / "scene_verdicts.npz", meta_json=np.frombuffer(json.dumps(out).encode(), np.uint8),
                        **arrays)
    print("scene_verdicts", [(r["id"], r["accepted"]) for r in out])


def traj_custom_obs():
    cfg = cfg_of(2, 5, assignment="fixed", seed=19)
    cfg.obs = ObsConfig(include_weather=False, k_road=20, k_vehicles=3, road_radius=12.5)
    eng = build_engine(cfg)
    rec = Recorder(full_obs_steps=range(1, 41))
    run_actions(eng, philox_actions(6, 40, 2, 5), rec)
    rec.save("traj_custom_obs")


def traj_reset():
    from drivegrid_bindings import EnvHandle
    eng = build_engine(cfg_of(2, 4, assignment="fixed", seed=23))
    env = EnvHandle(eng)
    acts = philox_actions(8, 30, 2, 4)
    rec = Recorder(full_obs_steps=(1, 30, 31, 60, 90))
    for t in range(30):
        env.step(acts[t].astype(np.float64))
    # snapshot of the engine output is taken through the recorder below
    obs_reset = env.reset()
    spawn_after_reset = eng.spawn_step.copy()
    step_after_reset = eng.step_count
    # overlapping starts through teleport_reset (new_starts) -> collision warmup
    starts = eng.start_xy.copy()
    starts[0, 1] = starts[0, 0] + np.array([1.0, 0.0])
    mask = np.zeros((2, 4), dtype=bool)
    mask[0] = True  # world 1 keeps the reset quirk (spawn_step = 30, age = -30)
    eng.teleport_reset(mask, new_starts=starts)
    zeros = np.zeros((60, 2, 4, 3), dtype=np.float32)
    zeros[:, 1] = acts[:30].repeat(2, axis=0)[:, 1]
    for t in range(60):
        out = eng.step(zeros[t].astype(np.float64))
        rec.add(t + 31, eng, out, zeros[t])
    rec.save("traj_reset", actions_pre=acts, obs_reset=obs_reset,
             spawn_after_reset=spawn_after_reset, step_after_reset=np.array(step_after_reset),
             starts=starts, mask=mask)


def event_actions(T, W, M):
    """Full throttle with a fixed per-agent steer; some agents brake hard
    mid-run.  Drives agents into goals, road edges and out past the 100 m
    drift limit so every event type fires."""
    steer = np.array([0.0, 0.08, -0.08, 0.3, -0.3, 0.02, -0.5, 0.15, 0.0, -0.15, 1.0,
                      -0.02, 0.6, 0.0, -1.0, 0.04])[:M]
    acts = np.zeros((T, W, M, 3), dtype=np.float32)
    acts[..., 0] = 1.0
    acts[..., 1] = steer[None, None, :] * (1.0 - 0.25 * (np.arange(W)[None, :, None] % 2))
    brake_rows = (np.arange(M) % 5 == 0)
    acts[100:160, :, brake_rows, 2] = 1.0
    acts[100:160, :, brake_rows, 0] = -1.0
    return acts


def traj_events():
    eng = build_engine(cfg_of(4, 16, seed=31))
    rec = Recorder(full_obs_steps=(1, 150, 420))
    run_actions(eng, event_actions(420, 4, 16), rec)
    rec.save("traj_events")


def traj_events_inv():
    eng = build_engine(cfg_of(4, 16, seed=31, invincible=True))
    rec = Recorder(full_obs_steps=(1, 150, 420))
    run_actions(eng, event_actions(420, 4, 16), rec)
    rec.save("traj_events_inv")


def _drac_record(name, eng, acts):
    """Engine.run_episode(record=True) -> pairwise_drac per logged step and
    episode_metrics over the log, exactly as the reference's eval does."""
    from drivegrid.metrics import episode_metrics, pairwise_drac

    it = iter(range(len(acts)))
    log = eng.run_episode(lambda obs: acts[next(it)].astype(np.float64), record=True,
                          max_steps=len(acts))
    per = {k: [] for k in ("x", "y", "yaw", "v_x", "v_y", "alive_pre", "drac", "goal", "collision")}
    for rec in log.steps:
        st = rec["state"]
        c, s = np.cos(st["yaw"]), np.sin(st["yaw"])
        vel = np.stack([st["v_x"] * c - st["v_y"] * s, st["v_x"] * s + st["v_y"] * c], axis=-1)
        pos = np.stack([st["x"], st["y"]], axis=-1)
        per["drac"].append(pairwise_drac(pos, st["yaw"], vel, eng.r_hull, eng.d_hull, rec["alive_pre"]))
        for k in ("x", "y", "yaw", "v_x", "v_y"):
            per[k].append(st[k])
        per["alive_pre"].append(rec["alive_pre"])
        per["goal"].append(rec["events"]["goal"])
        per["collision"].append(rec["events"]["collision"])
    em = episode_metrics(log, eng.valid, eng.length, eng.width)
    np.savez_compressed(
        OUT / f"{name}.npz", actions=acts[:len(log.steps)], r_hull=eng.r_hull, d_hull=eng.d_hull,
        valid=eng.valid, length=eng.length, width=eng.width,
        per_agent_max_drac=em.per_agent_max_drac, sr=em.sr, cr=em.cr,
        mean_max_drac=em.mean_max_drac, goals=em.goals, collisions=em.collisions,
        **{"step_" + k: np.stack(v) for k, v in per.items()})
    print(name, len(log.steps), "steps", em.to_dict())


def drac_wet():
    from drivegrid.config import load_scene_pool
    from drivegrid.engine import Engine, SimConfig
    from drivegrid.world import build_world_batch

    W, M = 12, 16
    cfg = cfg_of(W, M, seed=5)
    pool = load_scene_pool(cfg.scene_factory)
    worlds, assignment = build_world_batch(pool, W, mode="random_fill", seed=5)
    eng = Engine(worlds, pool, assignment, wet_frictions(W), SimConfig(num_envs=W, num_agents=M, seed=5))
    acts = philox_actions(9, 80, W, M)
    acts[..., 0] = np.abs(acts[..., 0])
    _drac_record("drac_wet", eng, acts)


def drac_events():
    eng = build_engine(cfg_of(4, 16, seed=31))
    _drac_record("drac_events", eng, event_actions(420, 4, 16))


def traj_timeout():
    eng = build_engine(cfg_of(2, 16, seed=17, episode_len=25))
    pol = LaneFollower(obs_config=eng.obs_config)
    rec = Recorder(full_obs_steps=(1, 25, 26, 40))
    obs = eng.observe()
    for t in range(40):
        a = pol(obs)
        out = eng.step(a)
        rec.add(t + 1, eng, out, a)
        obs = out.obs
    rec.save("traj_timeout")


def traj_forge():
    """Worlds round-tripped through the binary export (world.py:199-236): the
    engine runs on the float32-rounded imported geometry.  The export's bytes
    are pinned by their sha256."""
    import hashlib
    import tempfile

    from drivegrid.config import load_scene_pool, sample_weather
    from drivegrid.engine import Engine
    from drivegrid.vehicle import VehicleParams
    from drivegrid.world import build_world_batch, export_world_batch, import_world_batch
    from drivegrid.engine import SimConfig
    cfg = cfg_of(6, 16, seed=23)
    pool = load_scene_pool(cfg.scene_factory)
    built, assignment = build_world_batch(pool, 6, mode="random_fill", seed=23)
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "worlds.bin"
        export_world_batch(built, path)
        blob = path.read_bytes()
        worlds = import_world_batch(path)
    frictions = [assign_friction(s, h) for s, h in sample_weather(cfg.weather, 6, 23)]
    sim = SimConfig(num_envs=6, num_agents=16, seed=23)
    eng = Engine(worlds, pool, assignment, frictions, sim, obs_config=cfg.obs, reward_config=cfg.reward,
                 params=VehicleParams(), bicycle=cfg.bicycle)
    pol = LaneFollower(obs_config=eng.obs_config)
    rec = Recorder(full_obs_steps=(1, 40))
    obs = eng.observe()
    for t in range(40):
        a = pol(obs)
        out = eng.step(a)
        rec.add(t + 1, eng, out, a)
        obs = out.obs
    rec.save("traj_forge", export_sha256=np.frombuffer(hashlib.sha256(blob).digest(), dtype=np.uint8),
             export_nbytes=np.int64(len(blob)))


WEATHER_CASES = ((0.5, {"AC": 0.2, "SMA": 0.3, "OGFC": 0.5}, 0.1, 0.8, "AC", 7),
                 (1.0, {"AC": 0.0, "SMA": 2.0, "OGFC": 1.0}, 0.3, 0.3, "SMA", 11),
                 (0.25, {"OGFC": 1.0}, 0.05, 1.5, "OGFC", 42))


def weather_sampling():
    """sample_weather (config.py:141-157) for three weather configs x 64 worlds,
    and the engine's per-world mu / weather token under the first one."""
    from drivegrid.config import WeatherConfig, sample_weather
    out = {}
    for i, (wet, probs, fmin, fmax, dry, seed) in enumerate(WEATHER_CASES):
        cfg = WeatherConfig(wet_fraction=wet, surface_probs=probs, film_min_mm=fmin, film_max_mm=fmax,
                            dry_surface=dry)
        draws = sample_weather(cfg, 64, seed)
        out[f"c{i}_surface"] = np.array([SURFACE_ORDER.index(s) for s, _ in draws])
        out[f"c{i}_film"] = np.array([h for _, h in draws])
    cfg = cfg_of(16, 4, seed=7)
    cfg.weather.wet_fraction, cfg.weather.surface_probs = 0.5, dict(WEATHER_CASES[0][1])
    eng = build_engine(cfg)
    out["engine_mu_eff"], out["engine_weather"] = eng.mu_eff, eng.weather
    np.savez_compressed(OUT / "weather_sampling.npz", **out)
    print("weather_sampling", [int((out[f"c{i}_film"] > 0).sum()) for i in range(3)], "wet worlds")


GOAL_CASES = ((8, 29, 15.0, 60.0), (6, 31, 25.0, 25.0), (4, 37, 5000.0, 5000.0))


def goals_random():
    """eval.random_goals (config.py:222-278): goals before / after the
    resampling for three (W, seed, goal_min_m, goal_max_m) cases."""
    arrays = {}
    for i, (W, seed, lo, hi) in enumerate(GOAL_CASES):
        cfg = cfg_of(W, 16, seed=seed)
        before = build_engine(cfg)
        cfg.eval.random_goals, cfg.eval.goal_min_m, cfg.eval.goal_max_m = True, lo, hi
        after = build_engine(cfg)
        arrays[f"c{i}_start"] = after.start_xy
        arrays[f"c{i}_valid"] = after.valid
        arrays[f"c{i}_before"] = before.goal_xy
        arrays[f"c{i}_after"] = after.goal_xy
        print("goals_random", i, int((before.goal_xy != after.goal_xy).any(axis=-1).sum()), "goals moved")
    np.savez_compressed(OUT / "goals_random.npz", cases=np.array(GOAL_CASES), **arrays)


def _world_arrays(eng):
    """Every per-world init table of a reference engine (world.py:148-194,
    engine.py:176-253, config.py:236-278), canonical dtypes."""
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
    for k in vh.STATE_FIELDS:
        out["state_" + k] = eng.state[k]
    return out


def _canon(a):
    a = np.asarray(a)
    if a.dtype.kind == "f":
        a = a.astype(np.float64)
    elif a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return np.ascontiguousarray(a)


def worlds_4096():
    """On-device world construction pins at the scale it is for:
    sha256 of every init table of the reference's build_engine at 4096x16
    (default pool), with and without eval.random_goals (15-60 m)."""
    import hashlib
    arrays = {}
    for tag, goals in (("plain", False), ("goals", True)):
        cfg = cfg_of(4096, 16)
        if goals:
            cfg.eval.random_goals, cfg.eval.goal_min_m, cfg.eval.goal_max_m = True, 15.0, 60.0
        eng = build_engine(cfg)
        for k, v in _world_arrays(eng).items():
            c = _canon(v)
            arrays[f"{tag}__{k}__sha"] = np.frombuffer(hashlib.sha256(c.tobytes()).hexdigest().encode(), np.uint8)
            arrays[f"{tag}__{k}__shape"] = np.array(c.shape, dtype=np.int64)
        arrays[f"{tag}__goal_xy_head"] = eng.goal_xy[:64]
    np.savez_compressed(OUT / "worlds_4096.npz", **arrays)
    print("worlds_4096", len(arrays))


def worlds_cases():
    """The scene_cases pool (crowd > cap, edge-only scene without lanes, far goals,
    off-centre, elevated) through the reference's build_engine at 29 worlds:
    full init tables, with random goals (10-50 m; the lane-less scene draws none)."""
    import types

    from drivegrid import scenario as sc
    from drivegrid import synth
    from scene_cases import scene_specs
    mod = types.SimpleNamespace(Polyline=sc.Polyline, AgentRecord=sc.AgentRecord, ScenarioSpec=sc.ScenarioSpec,
                                straight_scene=synth.straight_scene, crossroads_scene=synth.crossroads_scene,
                                two_level_scene=synth.two_level_scene, shift_scenario=sc.shift_scenario)
    pool = [p for p in map(prepare_scene, scene_specs(mod)) if p is not None]
    arrays = {}
    for tag, goals in (("plain", False), ("goals", True)):
        cfg = cfg_of(29, 16, seed=7)
        if goals:
            cfg.eval.random_goals, cfg.eval.goal_min_m, cfg.eval.goal_max_m = True, 10.0, 50.0
        eng = build_engine(cfg, scenes=pool)
        for k, v in _world_arrays(eng).items():
            arrays[f"{tag}__{k}"] = _canon(v)
    np.savez_compressed(OUT / "worlds_cases.npz", **arrays)
    print("worlds_cases", len(pool), "scenes")


DENSE_LANES = tuple(float(x) for x in np.round(np.arange(-9.0, 9.01, 0.25), 2))


def traj_dense():
    """73 lanes 0.25 m apart: most agents see more than K_road = 350 road
    candidates, so the first-350-by-segment-index truncation is exercised."""
    scene = prepare_scene(straight_scene("dense", lane_offsets=DENSE_LANES, agent_count=8, agent_gap=15.0,
                                         goal_dist=40.0))
    eng = build_engine(cfg_of(2, 8, seed=3), scenes=[scene])
    pol = LaneFollower(obs_config=eng.obs_config)
    rec = Recorder(full_obs_steps=(1, 30))
    obs = eng.observe()
    for t in range(30):
        a = pol(obs)
        out = eng.step(a)
        rec.add(t + 1, eng, out, a)
        obs = out.obs
    rec.save("traj_dense")


def traj_sparse():
    scene = prepare_scene(straight_scene(agent_count=2, goal_dist=40.0))
    eng = build_engine(cfg_of(3, 4, seed=13), scenes=[scene])
    rec = Recorder(full_obs_steps=(1, 30, 60))
    run_actions(eng, philox_actions(12, 60, 3, 4), rec)
    rec.save("traj_sparse", valid=eng.valid)


class _NumpySpy:
    """Stands in for ``np`` inside drivegrid.observation / drivegrid.rewards and
    records the reference's own integer decisions: the stable argsorts of
    road_context (observation.py:96) and neighbor_features_batch
    (observation.py:246), and nearest_lane's argmin (rewards.py:94)."""

    def __init__(self):
        self.calls = []

    def __getattr__(self, name):
        return getattr(np, name)

    def argsort(self, a, *args, **kw):
        r = np.argsort(a, *args, **kw)
        self.calls.append((sys._getframe(1).f_code.co_name, "argsort", np.array(a), r))
        return r

    def argmin(self, a, *args, **kw):
        r = np.argmin(a, *args, **kw)
        self.calls.append((sys._getframe(1).f_code.co_name, "argmin", np.array(a), r))
        return r


def _index_record(spy, take_road, take_veh):
    """The step's calls -> (lane, road, road_n, veh, veh_n) like the kernel's
    index_out record (-1 for no lane)."""
    by = {name: (a, r) for name, _, a, r in spy.calls}
    not_cand, order = by["road_context"]
    road_n = np.minimum((~not_cand).sum(axis=-1), take_road)
    dist, sel = by["neighbor_features_batch"]
    sel = sel[..., :take_veh]
    veh_n = np.isfinite(np.take_along_axis(dist, sel, axis=-1)).sum(axis=-1)
    d2, k = by["nearest_lane"]
    best = np.take_along_axis(d2, k[..., None], axis=-1)[..., 0]
    lane = np.where(np.isfinite(best), k, -1)
    return lane, order[..., :take_road], road_n, sel, veh_n


def index_pins():
    """Integer decisions of the reference step (nearest-lane index, road slot
    -> segment map, neighbour order) captured from the reference's own
    argsort / argmin calls, serial engine (one world chunk per call)."""
    import drivegrid.observation as obs_mod
    import drivegrid.rewards as rw_mod
    spy = _NumpySpy()
    saved = obs_mod.np, rw_mod.np
    obs_mod.np, rw_mod.np = spy, spy
    try:
        for name, steps in (("traj_events", 160), ("traj_pool", 60)):
            if name == "traj_events":
                cfg = cfg_of(4, 16, seed=31)
                acts = event_actions(steps, 4, 16)
            else:
                cfg = cfg_of(4, 16)
                acts = None
            cfg.env.num_workers = 1
            eng = build_engine(cfg)
            take_road = min(eng.obs_config.k_road, eng.seg_mid.shape[-2])
            take_veh = min(eng.obs_config.k_vehicles, 16)
            pol = LaneFollower(obs_config=eng.obs_config)
            obs = eng.observe()
            rows = {k: [] for k in ("lane", "road", "road_n", "veh", "veh_n", "actions")}
            for t in range(steps):
                a = pol(obs) if acts is None else acts[t].astype(np.float64)
                alive_pre = eng.alive.copy()
                spy.calls.clear()
                out = eng.step(a)
                lane, road, road_n, veh, veh_n = _index_record(spy, take_road, take_veh)
                rows["lane"].append(np.where(alive_pre, lane, -1))
                rows["road"].append(road.astype(np.int16))
                rows["road_n"].append(road_n)
                rows["veh"].append(veh.astype(np.int8))
                rows["veh_n"].append(veh_n)
                rows["actions"].append(a)
                obs = out.obs
            np.savez_compressed(OUT / f"{name}_indices.npz", **{k: np.stack(v) for k, v in rows.items()})
            print(f"{name}_indices", steps, "steps")
    finally:
        obs_mod.np, rw_mod.np = saved


def sysid():
    import json
    from drivegrid import sysid as S
    from drivegrid.vehicle import VehicleParams, params_to_vector

    base = VehicleParams()
    lo, hi = S.default_bounds(base)
    rng = np.random.Generator(np.random.Philox(77))
    vectors = lo + (hi - lo) * rng.uniform(0.1, 0.9, (6, lo.size))
    vectors[0] = params_to_vector(base)
    teacher = VehicleParams(tau_drive_max=700.0, lambda_lat=120.0, kp_steer=1700.0, f_lat_wet=0.85)
    mans = {sc: S.generate_maneuvers(sc) for sc in (1.0, 0.2, 0.1)}
    pick, seen = [], set()
    for m in mans[1.0]:
        if m.kind not in seen:
            seen.add(m.kind)
            pick.append(m)
    batch = S.ParamBatch(base, vectors)
    tbatch = S.ParamBatch(teacher, params_to_vector(teacher)[None, :])
    arrays = {"vectors": vectors, "lo": lo, "hi": hi, "teacher": params_to_vector(teacher)}
    for i, m in enumerate(pick):
        st = S.rollout_channels(batch, m)
        te = S.rollout_channels(tbatch, m)
        for k, v in st.items():
            arrays[f"m{i}_{k}"] = v
            arrays[f"m{i}_teacher_{k}"] = te[k]
        arrays[f"m{i}_loss"] = S.sysid_loss(st, te)
    cem = S.CEMConfig(population=8, total_trials=40)
    res = S.run_cem(teacher, cem, scale=0.1, seed=3)
    meta = {
        "maneuvers": {str(sc): [[m.id, m.tier, m.kind, m.duration, m.params] for m in ms]
                      for sc, ms in mans.items()},
        "picked": [m.id for m in pick],
        "run_cem": res.to_dict(),
        "run_cem_args": {"population": 8, "total_trials": 40, "scale": 0.1, "seed": 3},
    }
    arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "sysid.npz", **arrays)
    print("sysid", len(pick), "maneuver kinds; run_cem best", res.stages[-1]["best_loss"])


if __name__ == "__main__":
    which = sys.argv[1:] or ["init_default", "friction", "friction_table", "traj_c1", "traj_pool", "traj_wet",
                             "traj_bicycle", "traj_custom_obs", "traj_reset", "traj_events",
                             "traj_events_inv", "drac_wet", "drac_events", "sysid", "traj_sparse", "traj_timeout", "traj_forge", "goals_random", "weather_sampling", "traj_dense", "traj_obs_min", "traj_no_edges", "scene_verdicts", "index_pins", "worlds_4096", "worlds_cases"]
    for name in which:
        globals()[name]()
