"""GPU kernel vs CPU oracle, on the same host-built tables and actions.

Bar (BASELINE north star): integer / boolean outputs (dones, events, reason,
alive, road-candidate counts, neighbour counts) bit-exact; float state,
observations and rewards within 1e-4 relative.  The kernel computes in
float64 with the reference's operation order, so the asserted tolerances
below are far tighter than that bar (state rtol 1e-9, obs 2 float32 ulp);
the observed maxima are printed for the record.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from cases import TRAJ_CASES, case_inputs, cfg_of
from oracle import OracleEngine
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.engine import Engine
from paper_2605_08528_b200.params import EVENT_TYPES, STATE_FIELDS
from paper_2605_08528_b200.policies import LaneFollower

pytestmark = pytest.mark.gpu

F64_RTOL, F64_ATOL = 1e-9, 1e-9
OBS_RTOL, OBS_ATOL = 1e-6, 1e-6


class Dev:
    """Running maxima of the float deviations."""

    def __init__(self):
        self.max = {}

    def f(self, name, got, want, rtol=F64_RTOL, atol=F64_ATOL):
        got = np.asarray(got, dtype=np.float64)
        want = np.asarray(want, dtype=np.float64)
        both = np.isfinite(got) & np.isfinite(want)
        assert np.array_equal(np.isfinite(got), np.isfinite(want)), f"{name}: finiteness differs"
        assert np.array_equal(got[~both], want[~both]), f"{name}: non-finite values differ"
        d = np.abs(got[both] - want[both])
        if d.size:
            self.max[name] = max(self.max.get(name, 0.0), float(d.max()))
        np.testing.assert_allclose(got[both], want[both], rtol=rtol, atol=atol, err_msg=name)


def obs_structure(obs, oc):
    """Integer structure of an observation batch: road candidates (type
    column non-zero) and valid neighbours (length column non-zero)."""
    road = obs[..., oc.ego_dim:oc.ego_dim + 5 * oc.k_road].reshape(obs.shape[:-1] + (oc.k_road, 5))
    veh = obs[..., oc.ego_dim + 5 * oc.k_road:].reshape(obs.shape[:-1] + (oc.k_vehicles, 7))
    return (road[..., 2] != 0).sum(-1), (veh[..., 2] != 0).sum(-1)


def compare(dev: Dev, t, g, o, oc):
    ctx = f"step {t}"
    for name in ("dones",):
        assert np.array_equal(np.asarray(getattr(g, name)), np.asarray(getattr(o, name))), f"{ctx} {name}"
    for k in EVENT_TYPES:
        assert np.array_equal(g.events[k], o.events[k]), f"{ctx} event {k}"
    for k in ("alive", "alive_pre", "reason"):
        assert np.array_equal(np.asarray(g.info[k]), np.asarray(o.info[k])), f"{ctx} {k}"
    gs, os_ = obs_structure(g.obs, oc), obs_structure(o.obs, oc)
    assert np.array_equal(gs[0], os_[0]), f"{ctx} road candidate counts"
    assert np.array_equal(gs[1], os_[1]), f"{ctx} neighbour counts"
    dev.f("rewards", g.rewards, o.rewards)
    dev.f("ttc_min", g.info["ttc_min"], o.info["ttc_min"])
    for k in g.info["reward_terms"]:
        dev.f(f"term_{k}", g.info["reward_terms"][k], o.info["reward_terms"][k])
    for k in STATE_FIELDS:
        dev.f(f"snap_{k}", g.info["state"][k], o.info["state"][k], rtol=F64_RTOL, atol=1e-9)
    dev.f("obs", g.obs, o.obs, rtol=OBS_RTOL, atol=OBS_ATOL)


VARIANTS = [(n, True, None, 0) for n in TRAJ_CASES] + [(n, True, None, 1) for n in TRAJ_CASES] + [
    ("traj_events", False, 3, 0), ("traj_wet", True, 16, 0), ("traj_pool", False, 1, 0),
    ("traj_events_inv", True, 5, 0), ("traj_events", False, 8, 1), ("traj_wet", False, 2, 1),
    ("traj_dense", False, 4, 0), ("traj_dense", True, 2, 1)]


@pytest.mark.parametrize("name", ["traj_events", "traj_wet", "traj_pool"])
def test_global_geometry_path_is_bit_identical(name, device):
    """Per-world blobs translated on the host (the path of scenes too large for
    shared memory) give exactly the outputs of the split kernels adding the
    grid offset on the fly, and match the oracle like every other path."""
    case = case_inputs(name)
    a = Engine(**case.inputs.as_kwargs(), device=device, launch_mode=1)
    b = Engine(**case.inputs.as_kwargs(), device=device, geometry_global=True)
    assert b.geometry_global and not a.geometry_global
    pol = LaneFollower(obs_config=a.obs_config)
    obs = a.observe()
    assert np.array_equal(obs, b.observe())
    for t in range(min(case.steps, 120)):
        act = pol(obs) if case.actions is None else case.actions[t].astype(np.float64)
        oa, ob = a.step(act), b.step(act)
        assert np.array_equal(oa.obs, ob.obs) and np.array_equal(oa.rewards, ob.rewards)
        assert np.array_equal(oa.dones, ob.dones) and np.array_equal(oa.info["reason"], ob.info["reason"])
        obs = oa.obs
    assert all(np.array_equal(a.state[k], b.state[k]) for k in STATE_FIELDS)


def test_global_geometry_rollout_loops_ticks(device):
    """A multi-tick rollout on a global-geometry engine (one split launch per
    tick) equals the same rollout on the fused engine."""
    case = case_inputs("traj_pool")
    a = Engine(**case.inputs.as_kwargs(), device=device)
    b = Engine(**case.inputs.as_kwargs(), device=device, geometry_global=True)
    a0 = a.lane_follower(a.observe_device())
    ra = a.rollout(a0.clone(), ticks=24, policy="lane_follower", autoreset=True)
    rb = b.rollout(a0.clone(), ticks=24, policy="lane_follower", autoreset=True)
    for k in ("obs", "rewards", "dones"):
        assert torch.allclose(getattr(ra, k).double(), getattr(rb, k).double(), rtol=1e-9, atol=1e-9), k


@pytest.mark.parametrize("mode", [0, 2])
def test_global_geometry_fused_variants(mode, device):
    """The fused kernel's global-geometry variants (kGeoGlobal: geometry read in
    place, multi-tick launches) on the dense scene give exactly the split
    kernels' outputs, tick by tick and over a 12-tick rollout launch."""
    case = case_inputs("traj_dense")
    a = Engine(**case.inputs.as_kwargs(), device=device)                       # split
    b = Engine(**case.inputs.as_kwargs(), device=device, launch_mode=mode)     # fused, global geometry
    assert a.geometry_global and b.geometry_global and b.launch_shape()["mode"] != "split"
    pol = LaneFollower(obs_config=a.obs_config)
    obs = a.observe()
    assert np.array_equal(obs, b.observe())
    for t in range(6):
        oa, ob = a.step(pol(obs)), b.step(pol(obs))
        assert np.array_equal(oa.obs, ob.obs) and np.array_equal(oa.rewards, ob.rewards)
        assert np.array_equal(oa.dones, ob.dones)
        obs = oa.obs
    a0 = a.lane_follower(a.observe_device())
    ra = a.rollout(a0.clone(), ticks=12, policy="lane_follower", autoreset=True)
    rb = b.rollout(a0.clone(), ticks=12, policy="lane_follower", autoreset=True)
    assert torch.equal(ra.obs, rb.obs) and torch.equal(ra.rewards, rb.rewards)
    assert all(np.array_equal(a.state[k], b.state[k]) for k in STATE_FIELDS)


def test_oversized_scene_runs_from_global_memory(device):
    case = case_inputs("traj_dense")
    eng = Engine(**case.inputs.as_kwargs(), device=device)
    assert eng.geometry_global
    with pytest.raises(Exception, match="shared memory"):
        Engine(**case.inputs.as_kwargs(), device=device, geometry_global=False)


@pytest.mark.parametrize("name,spatial,warps,mode", VARIANTS,
                         ids=[f"{n}-{'idx' if s else 'scan'}-w{w}-{'split' if m else 'fused'}"
                              for n, s, w, m in VARIANTS])
def test_trajectory_parity(name, spatial, warps, mode, device):
    """Launch mode/shape and the spatial index are performance knobs: every
    variant must reproduce the oracle."""
    case = case_inputs(name)
    gpu = Engine(**case.inputs.as_kwargs(), device=device, spatial_index=spatial,
                 warps_per_world=warps, launch_mode=mode)
    ora = OracleEngine(**case.inputs.as_kwargs())
    dev = Dev()
    dev.f("obs0", gpu.observe(), ora.observe(), rtol=OBS_RTOL, atol=OBS_ATOL)
    pol = LaneFollower(obs_config=ora.obs_config)
    obs = ora.observe()
    for t in range(case.steps):
        # teacher forcing for the closed-loop case: both step the oracle's action
        a = pol(obs) if case.actions is None else case.actions[t].astype(np.float64)
        o = ora.step(a)
        g = gpu.step(a)
        compare(dev, t + 1, g, o, ora.obs_config)
        obs = o.obs
    st = gpu.state
    for k in STATE_FIELDS:
        dev.f(f"state_{k}", st[k], ora.state[k])
    assert np.array_equal(gpu.reason, ora.reason)
    assert np.array_equal(gpu.alive, ora.alive)
    for k in EVENT_TYPES:
        assert np.array_equal(gpu.event_seen[k], ora.event_seen[k])
    print(f"\n[{name}] max |gpu - oracle|:", {k: f"{v:.2e}" for k, v in sorted(dev.max.items())})


@pytest.mark.parametrize("mode", [0, 1])
def test_event_counters_match_oracle(mode, device):
    """Device-accumulated per-world counters (events + alive agent-ticks)
    equal the host tally of the oracle's outputs."""
    case = case_inputs("traj_events")
    gpu = Engine(**case.inputs.as_kwargs(), device=device, launch_mode=mode)
    ora = OracleEngine(**case.inputs.as_kwargs())
    W = case.inputs.sim.num_envs
    counts = torch.zeros((W, 5), dtype=torch.int32, device=device)
    want = np.zeros((W, 5), dtype=np.int64)
    bufs = gpu.new_step_buffers()
    for t in range(case.steps):
        a = case.actions[t].astype(np.float64)
        o = ora.step(a)
        for i, k in enumerate(EVENT_TYPES):
            want[:, i] += o.events[k].sum(axis=1)
        want[:, 4] += o.info["alive_pre"].sum(axis=1)
        gpu.launch_step(torch.from_numpy(a).to(device), bufs, event_counts=counts)
    assert np.array_equal(counts.cpu().numpy(), want)
    assert want[:, :4].sum() > 0


def test_default_256x16_lane_follower_parity(device):
    """The headline shape (256 worlds x 16 agents, default pool, seed 42),
    LaneFollower closed loop, teacher-forced on the oracle's observations."""
    inp = C.build_inputs(C.RootConfig())
    gpu = Engine(**inp.as_kwargs(), device=device)
    ora = OracleEngine(**inp.as_kwargs(), num_workers=8)
    pol = LaneFollower(obs_config=ora.obs_config)
    dev = Dev()
    obs = ora.observe()
    for t in range(40):
        a = pol(obs)
        o = ora.step(a)
        g = gpu.step(a)
        compare(dev, t + 1, g, o, ora.obs_config)
        obs = o.obs
    print("\n[256x16] max |gpu - oracle|:", {k: f"{v:.2e}" for k, v in sorted(dev.max.items())})


def test_device_path_matches_host_path(device):
    """torch CUDA actions in -> CUDA outputs equal to the numpy path's."""
    inp = C.build_inputs(cfg_of(8, 16, seed=3))
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    g = np.random.Generator(np.random.Philox(1))
    for _ in range(20):
        act = g.uniform(-1, 1, (8, 16, 3)).astype(np.float32)
        oa = a.step(act.astype(np.float64))
        ob = b.step(torch.from_numpy(act).to(device))
        assert np.array_equal(oa.obs, ob.obs.cpu().numpy())
        assert np.array_equal(oa.rewards, ob.rewards.cpu().numpy())
        assert np.array_equal(oa.dones, ob.dones.cpu().numpy())
        for k in EVENT_TYPES:
            assert np.array_equal(oa.events[k], ob.events[k].cpu().numpy())


def test_device_lane_follower_equals_host_policy(device):
    inp = C.build_inputs(cfg_of(16, 16, seed=9))
    eng = Engine(**inp.as_kwargs(), device=device)
    pol = LaneFollower(obs_config=eng.obs_config)
    obs_d = eng.observe_device()
    for _ in range(30):
        acts_d = eng.lane_follower(obs_d)
        host = pol(obs_d.cpu().numpy())
        assert np.array_equal(acts_d.cpu().numpy(), host)
        assert torch.equal(pol.on_device(eng, obs_d), acts_d)
        out = eng.step(acts_d)
        obs_d = out.obs


@pytest.mark.parametrize("mode", [0, 1])
def test_fused_policy_equals_policy_kernel_and_host(mode, device):
    """The LaneFollower fused into the step (next_actions) reproduces both the
    stand-alone device policy kernel and the numpy policy bit for bit."""
    inp = C.build_inputs(cfg_of(16, 16, seed=9))
    a = Engine(**inp.as_kwargs(), device=device, launch_mode=mode)
    b = Engine(**inp.as_kwargs(), device=device, launch_mode=mode)
    pol = LaneFollower(obs_config=a.obs_config)
    acts = [torch.empty((16, 16, 3), dtype=torch.float64, device=device) for _ in range(2)]
    obs_a = a.observe(as_numpy=False, next_actions=acts[0])
    obs_b = b.observe(as_numpy=False)
    assert torch.equal(obs_a, obs_b)
    ba, bb = a.new_step_buffers(), b.new_step_buffers()
    for t in range(40):
        cur, nxt = acts[t % 2], acts[(t + 1) % 2]
        ref = b.lane_follower(obs_b)
        assert torch.equal(cur, ref)
        assert np.array_equal(cur.cpu().numpy(), pol(obs_b.cpu().numpy()))
        a.launch_step(cur, ba, autoreset=True, next_actions=nxt)
        b.launch_step(ref, bb, autoreset=True)
        assert torch.equal(ba.obs, bb.obs)
        obs_b = bb.obs.clone()


@pytest.mark.parametrize("mode", [0, 1])
def test_fused_autoreset_equals_step_then_teleport(mode, device):
    inp = C.build_inputs(cfg_of(8, 16, seed=31))
    a = Engine(**inp.as_kwargs(), device=device, launch_mode=mode)
    b = Engine(**inp.as_kwargs(), device=device, launch_mode=mode)
    from cases import event_actions
    acts = event_actions(200, 8, 16)
    resets = 0
    for t in range(200):
        x = torch.from_numpy(acts[t]).to(device)
        oa = a.step(x, autoreset=True)
        ob = b.step(x)
        b.teleport_reset(ob.dones)
        resets += int(ob.dones.sum())
        assert torch.equal(oa.obs, ob.obs)
        assert torch.equal(oa.rewards, ob.rewards)
        assert torch.equal(oa.dones, ob.dones)
        assert torch.equal(a.state_tensor, b.state_tensor)
        assert np.array_equal(a.alive, b.alive) and np.array_equal(a.reason, b.reason)
        assert np.array_equal(a.spawn_step, b.spawn_step)
    assert resets > 0


def test_nonfinite_action_rejected_before_mutation(device):
    inp = C.build_inputs(cfg_of(2, 4, assignment="fixed"))
    eng = Engine(**inp.as_kwargs(), device=device)
    before = eng.state_tensor.clone()
    acts = np.zeros((2, 4, 3))
    acts[1, 2, 0] = np.nan
    with pytest.raises(ValueError, match="world 1 agent 2"):
        eng.step(acts)
    with pytest.raises(ValueError, match="world 1 agent 2"):
        eng.step(torch.from_numpy(acts).to(device))
    assert torch.equal(before, eng.state_tensor)
    assert eng.step_count == 0
    with pytest.raises(ValueError, match="shape"):
        eng.step(np.zeros((2, 3, 3)))


@pytest.mark.parametrize("mode", [0, 1])
def test_device_guard_skips_bad_world(mode, device):
    """Without the host-side check the kernel still refuses to step a world
    whose actions are non-finite and reports the first bad element."""
    inp = C.build_inputs(cfg_of(3, 4, assignment="fixed"))
    eng = Engine(**inp.as_kwargs(), device=device, launch_mode=mode)
    st0 = eng.state_tensor.clone()
    acts = torch.zeros((3, 4, 3), dtype=torch.float64, device=device)
    acts[..., 0] = 1.0
    acts[2, 1, 2] = float("inf")
    bufs = eng.new_step_buffers()
    eng.launch_step(acts, bufs)
    with pytest.raises(ValueError, match="world 2 agent 1"):
        eng.raise_pending_error()
    st1 = eng.state_tensor
    assert torch.equal(st1[:, 2], st0[:, 2])          # bad world untouched
    assert not torch.equal(st1[:, 0], st0[:, 0])      # others stepped


def test_env_handle_reset_quirk_and_shapes(device):
    from paper_2605_08528_b200.bindings import EnvHandle
    g = np.load(__import__("cases").GOLDEN / "traj_reset.npz")
    inp = C.build_inputs(cfg_of(2, 4, assignment="fixed", seed=23))
    eng = Engine(**inp.as_kwargs(), device=device)
    env = EnvHandle(eng)
    assert env.shapes["obs"] == (2, 4, 1929)
    ora = OracleEngine(**inp.as_kwargs())
    for t in range(30):
        a = g["actions_pre"][t].astype(np.float64)
        env.step(a)
        ora.step(a)
    obs = env.reset()
    assert obs.dtype == np.float32
    np.testing.assert_allclose(obs, ora.env_reset(), rtol=OBS_RTOL, atol=OBS_ATOL)
    assert np.array_equal(eng.spawn_step, ora.spawn_step)   # stamped 30, then step_count = 0
    assert eng.step_count == 0
    eng.teleport_reset(g["mask"], new_starts=g["starts"])
    ora.teleport_reset(g["mask"], new_starts=g["starts"])
    dev = Dev()
    for i in range(60):
        a = g["actions"][i]
        compare(dev, i + 31, eng.step(a), ora.step(a), ora.obs_config)
    with pytest.raises(ValueError, match="shape"):
        env.step(np.zeros((2, 2, 3)))


def test_make_env_default_shapes(device):
    from paper_2605_08528_b200.bindings import make_env
    env = make_env(None, device=device)
    assert env.shapes["obs"] == (256, 16, 1929)
    obs = env.reset()
    assert obs.shape == (256, 16, 1929) and obs.dtype == np.float32
    with pytest.raises(FileNotFoundError):
        make_env("/nonexistent/config.yaml")


def test_state_get_set_through_the_c_abi(device):
    """dg_get_state / dg_set_state: a state saved after k steps and loaded back
    into a fresh engine reproduces the next steps (teacher forcing)."""
    inp = C.build_inputs(cfg_of(4, 16, seed=3))
    a = Engine(**inp.as_kwargs(), device=device)
    acts = np.random.Generator(np.random.Philox(1)).uniform(-1, 1, (12, 4, 16, 3))
    for t in range(6):
        a.step(acts[t])
    saved = torch.tensor(np.stack([a.state[k] for k in STATE_FIELDS]))
    b = Engine(**inp.as_kwargs(), device=device)
    b.load_state_tensor(saved.to(device))
    for k in ("alive", "reason", "event_seen", "spawn_step"):
        b.device_tables()[k].copy_(a.device_tables()[k])
    b.step_count = a.step_count
    for t in range(6, 12):
        oa, ob = a.step(acts[t]), b.step(acts[t])
        assert np.array_equal(oa.obs, ob.obs) and np.array_equal(oa.rewards, ob.rewards)
    for k in STATE_FIELDS:
        assert np.array_equal(a.state[k], b.state[k])


def test_random_goals_engine_parity(device):
    """config.build_engine with eval.random_goals: the GPU engine carries the
    reference's resampled goals (golden goals_random) and steps like the oracle
    driven to the same goals."""
    g = np.load(__import__("cases").GOLDEN / "goals_random.npz")
    W, seed, lo, hi = g["cases"][0]
    cfg = cfg_of(int(W), 16, seed=int(seed))
    cfg.eval.random_goals, cfg.eval.goal_min_m, cfg.eval.goal_max_m = True, float(lo), float(hi)
    gpu = C.build_engine(cfg, device=device)
    assert np.array_equal(gpu.goal_xy, g["c0_after"])
    ora = OracleEngine(**C.build_inputs(cfg).as_kwargs())
    ora.goal_xy = g["c0_after"].copy()
    dev = Dev()
    pol = LaneFollower(obs_config=ora.obs_config)
    obs = ora.observe()
    dev.f("obs0", gpu.observe(), obs, rtol=OBS_RTOL, atol=OBS_ATOL)
    for t in range(40):
        a = pol(obs)
        o = ora.step(a)
        compare(dev, t + 1, gpu.step(a), o, ora.obs_config)
        obs = o.obs
    assert np.array_equal(gpu.reason, ora.reason) and np.array_equal(gpu.alive, ora.alive)


@pytest.mark.parametrize("scene_id", ["crowd", "shifted", "hilly", "ramp"])
def test_scene_intake_cases_step_like_the_oracle(scene_id, device):
    """The synthetic intake specs (tests/golden/scene_cases.py: more agents
    than slots, an off-centre scene, an elevated one, a low ramp) stepped on
    the GPU against the oracle under the LaneFollower."""
    import sys
    import types

    from cases import GOLDEN
    from paper_2605_08528_b200 import scenes as S
    sys.path.insert(0, str(GOLDEN))
    from scene_cases import scene_specs
    mod = types.SimpleNamespace(Polyline=S.Polyline, AgentRecord=S.AgentRecord, ScenarioSpec=S.ScenarioSpec,
                                straight_scene=S.straight_scene, crossroads_scene=S.crossroads_scene,
                                two_level_scene=S.two_level_scene, shift_scenario=S.shift_scenario)
    spec = next(s for s in scene_specs(mod) if s.scenario_id == scene_id)
    inp = C.build_inputs(cfg_of(2, 16, seed=5), scenes=[S.prepare_scene(spec)])
    gpu = Engine(**inp.as_kwargs(), device=device)
    ora = OracleEngine(**inp.as_kwargs())
    dev = Dev()
    pol = LaneFollower(obs_config=ora.obs_config)
    obs = ora.observe()
    dev.f("obs0", gpu.observe(), obs, rtol=OBS_RTOL, atol=OBS_ATOL)
    for t in range(60):
        a = pol(obs)
        o = ora.step(a)
        compare(dev, t + 1, gpu.step(a), o, ora.obs_config)
        obs = o.obs
    assert np.array_equal(gpu.reason, ora.reason) and np.array_equal(gpu.alive, ora.alive)
