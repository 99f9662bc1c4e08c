"""Engine semantics on the GPU, one behaviour per test: the contract the
reference's own engine tests pin (pkg/tests/test_engine.py:18-292) -- slot
occupancy and parking, per-world friction, determinism, action validation,
goal payout and teleport, visibility of terminated agents, timeout, the
24-tick collision warm-up, teleport resets, episode logs, invincible mode --
restated against this package's Engine (the trajectory parity tests cover
the same paths value by value; these read as the reference's tests do)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.params import OFFSTAGE_X, REASON_GOAL, REASON_TIMEOUT
from paper_2605_08528_b200.policies import LaneFollower, ZeroPolicy
from paper_2605_08528_b200.scenes import prepare_scene, straight_scene

pytestmark = pytest.mark.gpu


def small_engine(device, num_envs=2, num_agents=4, mode="dynamic", scenes=None, seed=42, invincible=False,
                 episode_len=1500, wet=None):
    cfg = C.RootConfig()
    cfg.env.num_envs, cfg.env.num_agents_per_env = num_envs, num_agents
    cfg.env.dynamics_mode, cfg.env.episode_len = mode, episode_len
    cfg.eval.invincible, cfg.seed = invincible, seed
    cfg.scene_factory.assignment_mode = "fixed"
    if wet is not None:
        cfg.weather.wet_fraction, cfg.weather.surface_probs = 1.0, {wet[0]: 1.0}
        cfg.weather.film_min_mm = cfg.weather.film_max_mm = wet[1]
    if scenes is None:
        scenes = [prepare_scene(straight_scene(agent_count=num_agents, agent_gap=10.0, lane_offsets=(0.0, 4.0)))]
    return C.build_engine(cfg, scenes=scenes, device=device)


def _lone_runner(device, mode="dynamic", goal_dist=20.0):
    scene = prepare_scene(straight_scene(agent_count=1, goal_dist=goal_dist))
    return small_engine(device, 1, 1, mode=mode, scenes=[scene])


def _overlapping_pair(device, invincible=False):
    scene = prepare_scene(straight_scene(agent_count=2, agent_gap=30.0, goal_dist=40.0))
    eng = small_engine(device, 1, 2, scenes=[scene], invincible=invincible)
    starts = eng.start_xy.copy()
    starts[0, 1] = starts[0, 0] + np.array([1.0, 0.0])        # hulls overlap at spawn
    eng.teleport_reset(np.ones((1, 2), dtype=bool), new_starts=starts)
    return eng


def test_ragged_slots_are_parked_offstage(device):
    rich = prepare_scene(straight_scene("rich", agent_count=3, agent_gap=12.0))
    poor = prepare_scene(straight_scene("poor", agent_count=1))
    eng = small_engine(device, 2, 3, scenes=[rich, poor])
    assert np.array_equal(eng.alive, [[True, True, True], [True, False, False]])
    assert eng.state["x"][1, 1] == eng.worlds.grid_offsets[1, 0] + OFFSTAGE_X


def test_friction_is_per_world(device):
    eng = small_engine(device, 2, wet=("AC", 0.5))
    assert eng.mu_eff.shape == (2,)
    assert np.allclose(eng.weather[0], [0.5, 1, 0, 0])
    assert abs(eng.mu_eff[0] - min(eng.frictions[0].mu_static, 1.0)) < 1e-12


def test_same_seed_same_engine_same_trajectory(device):
    a, b = small_engine(device, seed=3), small_engine(device, seed=3)
    assert all(np.array_equal(a.state[k], b.state[k]) for k in a.state)
    assert np.array_equal(a.goal_xy, b.goal_xy)
    acts = np.random.Generator(np.random.Philox(77)).uniform(-1, 1, (40, 2, 4, 3))
    for t in range(40):
        oa, ob = a.step(acts[t]), b.step(acts[t])
        assert np.array_equal(oa.obs, ob.obs) and np.array_equal(oa.rewards, ob.rewards)
    assert all(np.array_equal(a.state[k], b.state[k]) for k in a.state)


def test_zero_actions_stay_put(device):
    eng = small_engine(device)
    before = eng.pos.copy()
    out = eng.step(np.zeros((2, 4, 3)))
    assert not out.dones.any() and np.abs(eng.pos - before).max() < 1e-9


def test_bad_actions_rejected(device):
    eng = small_engine(device)
    acts = np.zeros((2, 4, 3))
    acts[1, 2, 0] = np.nan
    with pytest.raises(ValueError, match="world 1 agent 2"):
        eng.step(acts)
    with pytest.raises(ValueError, match="shape"):
        eng.step(np.zeros((2, 3, 3)))


@pytest.mark.parametrize("mode", ["dynamic", "bicycle"])
def test_full_throttle_reaches_the_goal(mode, device):
    eng = _lone_runner(device, mode)
    acts = np.zeros((1, 1, 3))
    acts[..., 0] = 1.0
    for _ in range(1500):
        if eng.step(acts).dones.any():
            break
    assert eng.reason[0, 0] == REASON_GOAL and eng.step_count < 1500


def test_goal_pays_45_parks_and_then_pays_nothing(device):
    eng = _lone_runner(device)
    acts = np.zeros((1, 1, 3))
    acts[..., 0] = 1.0
    r_done = None
    for _ in range(1500):
        out = eng.step(acts)
        if out.dones[0, 0]:
            r_done = out.rewards[0, 0]
            break
    assert r_done is not None and abs(r_done - 45.0) < 5.0
    assert not eng.alive[0, 0]
    assert eng.state["x"][0, 0] == OFFSTAGE_X and eng.state["v_x"][0, 0] == 0.0
    out = eng.step(acts)
    assert out.rewards[0, 0] == 0.0 and not out.dones[0, 0]


def test_finished_agent_leaves_the_neighbour_block(device):
    scene = prepare_scene(straight_scene(agent_count=2, agent_gap=10.0, goal_dist=20.0))
    eng = small_engine(device, 1, 2, scenes=[scene])
    acts = np.zeros((1, 2, 3))
    acts[0, 1, 0] = 1.0                                        # only the lead car drives
    for _ in range(1500):
        eng.step(acts)
        if not eng.alive[0, 1]:
            break
    assert eng.reason[0, 1] == REASON_GOAL
    out = eng.step(np.zeros((1, 2, 3)))
    oc = eng.obs_config
    assert (out.obs[0, 0, oc.ego_dim + oc.k_road * 5:] == 0).all()


def test_timeout_reason_and_log_length(device):
    eng = small_engine(device, 1, 2, episode_len=30)
    log = eng.run_episode(ZeroPolicy(), record=True)
    assert len(log) == 30 and (eng.reason[eng.valid] == REASON_TIMEOUT).all()


def test_run_episode_stops_once_everyone_is_done(device):
    eng = _lone_runner(device)
    log = eng.run_episode(LaneFollower(throttle=1.0, obs_config=eng.obs_config), record=True)
    assert eng.reason[0, 0] == REASON_GOAL and len(log) == eng.step_count < 1500


def test_one_tick_is_four_physics_substeps(device):
    """A control tick = decimation (4) substeps of the 120 Hz single-track
    model on the clipped action, from the tick's starting state: the oracle's
    substep (oracle/stepper.py, vehicle.py:237-336) applied by hand gives the
    GPU's state to float64 rounding."""
    from oracle.stepper import decode, substep_dynamic
    eng = small_engine(device, 1, 1)
    acts = np.zeros((1, 1, 3))
    acts[..., 0] = 0.8
    manual = {k: v.copy() for k, v in eng.state.items()}
    eng.step(acts)
    for _ in range(eng.config.decimation):
        manual = substep_dynamic(manual, decode(acts), eng.mu_eff[:, None], eng.params, eng.config.physics_dt)
    for k in ("x", "v_x", "wheel_front"):
        assert abs(eng.state[k][0, 0] - manual[k][0, 0]) <= 1e-12 * max(1.0, abs(manual[k][0, 0])), k
    assert eng.state["v_x"][0, 0] > 0.0


def test_teleport_reset_restores_spawn_and_none_is_noop(device):
    eng = small_engine(device, seed=21)
    fresh = {k: v.copy() for k, v in eng.state.items()}
    before = {k: v.copy() for k, v in eng.state.items()}
    eng.teleport_reset(np.zeros((2, 4), dtype=bool))
    assert all(np.array_equal(eng.state[k], before[k]) for k in before)
    rng = np.random.Generator(np.random.Philox(2))
    for _ in range(20):
        eng.step(rng.uniform(-1, 1, (2, 4, 3)))
    eng.teleport_reset(np.ones((2, 4), dtype=bool))
    v = eng.valid
    assert all(np.array_equal(eng.state[k][v], fresh[k][v]) for k in fresh)
    assert np.array_equal(eng.alive, v) and (eng.spawn_step[v] == eng.step_count).all()


def test_collision_suppressed_for_exactly_24_ticks(device):
    eng = _overlapping_pair(device)
    hits = []
    for _ in range(30):
        hits.append(bool(eng.step(np.zeros((1, 2, 3))).events["collision"].any()))
        if hits[-1]:
            break
    assert hits.index(True) == 24 and not any(hits[:24])


def test_invincible_mode_latches_without_terminating(device):
    eng = _overlapping_pair(device, invincible=True)
    saw = False
    for _ in range(30):
        out = eng.step(np.zeros((1, 2, 3)))
        saw |= bool(out.events["collision"].any())
        assert not out.dones.any()
    assert saw and eng.alive.all() and eng.event_seen["collision"].any()


def test_episode_log_jsonl_and_60hz(device, tmp_path):
    eng = small_engine(device, 1, 2)
    log = eng.run_episode(LaneFollower(obs_config=eng.obs_config), record=True, max_steps=5)
    f = tmp_path / "traj.jsonl"
    log.to_jsonl(f)
    rows = [json.loads(line) for line in f.read_text().splitlines()]
    assert len(rows) == 5 * 2 and rows[0]["step"] == 1 and "reward" in rows[0] and "pose" in rows[0]
    assert rows[2]["pose"][0] == log.steps[1]["state"]["x"][0, 0]       # float64 survives JSON
    assert len(log.resample_60hz()) == 2 * len(log)


@pytest.mark.parametrize("quarter", [1, 2, 3])
def test_observations_are_rotation_equivariant(quarter, device):
    """The observation contract's equivariance (test_acceptance.py:140-186):
    the crossroads scene turned by a quarter / half / three-quarter turn
    (exact in float64, and the square scene box is invariant) yields the same
    body-frame observations, rewards and events under the same actions."""
    from paper_2605_08528_b200.scenes import AgentRecord, Polyline, ScenarioSpec, crossroads_scene
    c, s = {1: (0.0, 1.0), 2: (-1.0, 0.0), 3: (0.0, -1.0)}[quarter]

    def rot(x, y):
        return c * x - s * y, s * x + c * y

    base = crossroads_scene(agent_count=8)
    turned = ScenarioSpec(
        "turned",
        [Polyline(p.type_code, np.stack([*rot(p.points[:, 0], p.points[:, 1]), p.points[:, 2]], axis=1))
         for p in base.polylines],
        [AgentRecord(a.id, rot(*a.start), a.start_heading + quarter * np.pi / 2, rot(*a.goal), a.length, a.width)
         for a in base.agents])
    ea = small_engine(device, 1, 8, scenes=[prepare_scene(base)])
    eb = small_engine(device, 1, 8, scenes=[prepare_scene(turned)])
    pol = LaneFollower(obs_config=ea.obs_config)
    oa, ob = ea.observe(), eb.observe()
    assert np.allclose(oa, ob, rtol=1e-6, atol=1e-6)
    for _ in range(40):
        act = pol(oa)
        sa, sb = ea.step(act), eb.step(act)
        assert np.allclose(sa.obs, sb.obs, rtol=1e-6, atol=1e-6)
        assert np.allclose(sa.rewards, sb.rewards, rtol=1e-9, atol=1e-9)
        assert np.array_equal(sa.dones, sb.dones) and np.array_equal(sa.info["reason"], sb.info["reason"])
        oa = sa.obs


def test_phase_seconds_split_by_device_phase_cycles(device):
    """Engine.phase_seconds (engine.py:33, 342-395) on the GPU: the fused kernel
    counts device cycles per phase (DgStepIO.phase_cycles), the host books each
    step's wall time over the phases in that proportion -- every phase the step
    runs gets time, and the phases sum to the measured step time."""
    import time

    from paper_2605_08528_b200.params import PHASES
    from paper_2605_08528_b200.policies import LaneFollower
    eng = C.build_engine(C.RootConfig(), device=device)
    pol = LaneFollower(obs_config=eng.obs_config)
    obs = eng.observe()
    for _ in range(3):
        obs = eng.step(pol(obs), autoreset=True).obs
    eng.reset_phase_timers()
    t0 = time.perf_counter()
    acts = [pol(obs)]
    for _ in range(20):
        obs = eng.step(acts[-1], autoreset=True).obs
        acts.append(pol(obs))
    wall = time.perf_counter() - t0
    ph = eng.phase_seconds
    assert set(ph) == set(PHASES)
    for k in ("action", "physics", "observation", "reward_termination"):
        assert ph[k] > 0.0, k
    assert 0.3 * wall < sum(ph.values()) <= wall
    cyc = np.array(eng._phase_host)
    assert cyc[2] > cyc[1] > 0 and cyc[3] > 0          # observation > physics > 0 on the device
