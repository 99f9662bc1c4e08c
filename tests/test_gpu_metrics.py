"""Episode safety metrics on the GPU (a19: pairwise DRAC, SR / CR) against the
reference's own numbers (tests/golden/drac_*.npz, made by running
drivegrid.metrics) and against the CPU oracle (oracle/metrics.py).

Bar: goal / collision counts, SR, CR and the set of agents over the DRAC
threshold exact; DRAC values within 1e-9 relative (float64 in the reference's
operation order; only CUDA's cos/sin may differ from libm in the last ulp).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from cases import GOLDEN, case_inputs, cfg_of, wet_frictions
from oracle import OracleEngine
from oracle.metrics import aggregate as oracle_aggregate
from oracle.metrics import drac_of_snapshot
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200 import metrics as GM
from paper_2605_08528_b200.engine import Engine
from paper_2605_08528_b200.params import EVENT_TYPES

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-9, 1e-12


def golden_log(g):
    T = g["step_x"].shape[0]
    recs = []
    for t in range(T):
        recs.append({"state": {k: g["step_" + k][t] for k in ("x", "y", "yaw", "v_x", "v_y")},
                     "alive_pre": g["step_alive_pre"][t],
                     "events": {"goal": g["step_goal"][t], "collision": g["step_collision"][t]}})
    return recs


def check_metrics(m, g, threshold=3.4):
    assert m.goals == int(g["goals"]) and m.collisions == int(g["collisions"])
    assert m.valid_agents == int(g["valid"].sum())
    assert m.sr == float(g["sr"]) and m.cr == float(g["cr"])
    want = g["per_agent_max_drac"]
    np.testing.assert_allclose(m.per_agent_max_drac, want, rtol=RTOL, atol=ATOL)
    assert np.array_equal(m.per_agent_max_drac > threshold, want > threshold)
    np.testing.assert_allclose(m.mean_max_drac, float(g["mean_max_drac"]), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("name", ["drac_wet", "drac_events"])
def test_pairwise_drac_kernel_matches_reference(name, device):
    g = np.load(GOLDEN / f"{name}.npz")
    T = g["step_x"].shape[0]
    for t in range(0, T, max(1, T // 25)):
        x, y, yaw = g["step_x"][t], g["step_y"][t], g["step_yaw"][t]
        c, s = np.cos(yaw), np.sin(yaw)
        vel = np.stack([g["step_v_x"][t] * c - g["step_v_y"][t] * s,
                        g["step_v_x"][t] * s + g["step_v_y"][t] * c], axis=-1)
        got = GM.pairwise_drac(np.stack([x, y], -1), yaw, vel, g["r_hull"], g["d_hull"],
                               g["step_alive_pre"][t])
        np.testing.assert_allclose(got, g["step_drac"][t], rtol=RTOL, atol=ATOL, err_msg=f"step {t}")
        assert np.array_equal(got > 0, g["step_drac"][t] > 0)


@pytest.mark.parametrize("name", ["drac_wet", "drac_events"])
def test_episode_metrics_of_log_matches_reference(name, device):
    g = np.load(GOLDEN / f"{name}.npz")
    m = GM.episode_metrics(golden_log(g), g["valid"], g["length"], g["width"])
    check_metrics(m, g)


@pytest.mark.parametrize("name,mode,ticks", [("drac_wet", 0, 1), ("drac_wet", 1, 1), ("drac_events", 0, 1),
                                             ("drac_events", 1, 1), ("drac_wet", 0, 80),
                                             ("drac_events", 0, 140)])
def test_in_kernel_metrics_match_reference(name, mode, ticks, device):
    """track_episode_metrics: the step kernel accumulates what episode_metrics
    derives from a recorded log -- same numbers, no log."""
    g = np.load(GOLDEN / f"{name}.npz")
    case = case_inputs("traj_wet" if name == "drac_wet" else "traj_events")
    eng = Engine(**case.inputs.as_kwargs(), device=device, launch_mode=mode)
    eng.track_episode_metrics()
    acts = g["actions"].astype(np.float64)
    T = acts.shape[0]
    if ticks == 1:
        for t in range(T):
            out = eng.step(acts[t])
            if not out.info["alive"].any():
                break
    else:
        a = torch.as_tensor(acts, device=device)
        for t0 in range(0, T, ticks):
            eng.rollout(a[t0:t0 + ticks])
    check_metrics(eng.episode_metrics(), g)


def test_c3_wet_sweep_256x16_events_and_drac(device):
    """BASELINE configs[2]: 256 worlds x 16 agents, per-world friction sweep
    (AC / SMA / OGFC x water film 0..2 mm tiled over the worlds): events,
    dones and reasons bit-exact every step; per-agent peak DRAC and SR / CR
    against the oracle."""
    W, M, T = 256, 16, 48
    inp = C.build_inputs(cfg_of(W, M, seed=7))
    inp.frictions = wet_frictions(W)
    gpu = Engine(**inp.as_kwargs(), device=device)
    ora = OracleEngine(**inp.as_kwargs())
    assert np.array_equal(gpu.mu_eff, ora.mu_eff)
    assert len(np.unique(gpu.mu_eff)) >= 8          # the sweep really varies mu
    gpu.track_episode_metrics()
    rng = np.random.Generator(np.random.Philox(17))
    acts = rng.uniform(-1, 1, (T, W, M, 3)).astype(np.float32)
    acts[..., 0] = np.abs(acts[..., 0])
    mx = np.zeros((W, M))
    goal = np.zeros((W, M), dtype=bool)
    coll = np.zeros((W, M), dtype=bool)
    n_events = 0
    for t in range(T):
        a = acts[t].astype(np.float64)
        go, oo = gpu.step(a), ora.step(a)
        assert np.array_equal(go.dones, oo.dones), t
        for k in EVENT_TYPES:
            assert np.array_equal(go.events[k], oo.events[k]), (t, k)
            n_events += int(oo.events[k].sum())
        assert np.array_equal(go.info["reason"], oo.info["reason"]), t
        assert np.array_equal(go.info["alive"], oo.info["alive"]), t
        mx = np.maximum(mx, drac_of_snapshot(oo.info["state"], oo.info["alive_pre"], ora.r_hull, ora.d_hull))
        goal |= oo.events["goal"]
        coll |= oo.events["collision"]
    assert n_events > 0
    want = oracle_aggregate(goal, coll, mx, ora.valid)
    m = gpu.episode_metrics()
    assert (m.goals, m.collisions, m.valid_agents) == (want["goals"], want["collisions"], want["valid_agents"])
    np.testing.assert_allclose(m.per_agent_max_drac, mx, rtol=RTOL, atol=ATOL)
    assert np.array_equal(m.per_agent_max_drac > 3.4, mx > 3.4)
    assert (mx > 0).any()
    np.testing.assert_allclose(m.mean_max_drac, want["mean_max_drac"], rtol=RTOL, atol=ATOL)


def test_metrics_off_by_default_and_reset(device):
    case = case_inputs("traj_events")
    eng = Engine(**case.inputs.as_kwargs(), device=device)
    with pytest.raises(RuntimeError):
        eng.episode_metrics()
    eng.track_episode_metrics()
    for t in range(30):
        eng.step(case.actions[t].astype(np.float64))
    eng.reset_episode_metrics()
    m = eng.episode_metrics()
    assert m.goals == 0 and m.collisions == 0 and not m.per_agent_max_drac.any()


# ---- the reference's metrics unit contract (pkg/tests/test_metrics.py:14-110)
def _head_on_log(v_closing=8.0, gap=12.0):
    """One logged tick: agent 1 drives straight at agent 0 from ``gap`` m."""
    from paper_2605_08528_b200.engine import LOG_STATE_FIELDS, EpisodeLog
    st = {k: np.zeros((1, 2)) for k in LOG_STATE_FIELDS}
    st["x"][0, 0], st["v_x"][0, 1] = gap, v_closing
    log = EpisodeLog(control_dt=1 / 30)
    zero, alive = np.zeros((1, 2)), np.ones((1, 2), dtype=bool)
    log.append(1, st, np.zeros((1, 2, 3)), zero, {"total": zero}, {k: ~alive for k in EVENT_TYPES}, ~alive, alive,
               alive)
    return log


def test_hand_built_head_on_drac(device):
    log = _head_on_log()
    rec = log.steps[0]
    pos = np.stack([rec["state"]["x"], rec["state"]["y"]], axis=-1)
    vel = np.stack([rec["state"]["v_x"], rec["state"]["v_y"]], axis=-1)
    vals = GM.pairwise_drac(pos, rec["state"]["yaw"], vel, np.full((1, 2), 1.10), np.full((1, 2), 1.12),
                            rec["alive_pre"])
    hull_gap = 12.0 - 2 * 1.12 - 2 * 1.10
    assert np.allclose(vals[0], [64.0 / (2 * hull_gap)] * 2, rtol=1e-12)
    m = GM.episode_metrics(log, np.ones((1, 2), dtype=bool))
    assert (m.sr, m.cr, m.valid_agents) == (0.0, 0.0, 2)
    assert abs(m.mean_max_drac - 64.0 / (2 * (12.0 - 4.44))) < 1e-9


def test_everyone_reaching_the_goal_scores_sr_one(device):
    from paper_2605_08528_b200.policies import LaneFollower
    from paper_2605_08528_b200.scenes import prepare_scene, straight_scene
    cfg = cfg_of(1, 2, assignment="fixed")
    scene = prepare_scene(straight_scene(agent_count=2, agent_gap=12.0, goal_dist=20.0))
    eng = C.build_engine(cfg, scenes=[scene], device=device)
    log = eng.run_episode(LaneFollower(throttle=1.0, obs_config=eng.obs_config), record=True)
    m = GM.episode_metrics(log, eng.valid, eng.length, eng.width)
    assert m.sr == 1.0 and m.cr == 0.0


def test_measure_engine_report(device):
    from paper_2605_08528_b200.params import PHASES
    from paper_2605_08528_b200.policies import ZeroPolicy
    eng = Engine(**C.build_inputs(cfg_of(2, 2, assignment="fixed")).as_kwargs(), device=device)
    rep = GM.measure_engine(eng, ZeroPolicy(), steps=6, warmup=2)
    assert rep.casps > 0 and rep.steps == 6 and set(rep.phase_ms) == set(PHASES)
    assert all(v >= 0 for v in rep.phase_ms.values())
