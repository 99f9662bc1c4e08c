"""Persistent multi-tick launches (DgStepIO.ticks): a T-tick rollout in one
kernel launch must equal T separate step launches bit for bit -- every
per-tick output, the final state, the step counter and the episode counters
-- and therefore the oracle (env.py:48-65 called T times)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from cases import case_inputs, cfg_of, event_actions, philox_actions
from oracle import OracleEngine
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.engine import Engine
from paper_2605_08528_b200.params import EVENT_TYPES

from test_gpu_parity import Dev, compare

pytestmark = pytest.mark.gpu

OUT_VIEWS = ("rewards", "ttc_min", "terms", "snapshot", "events", "dones", "reason", "alive", "alive_pre")


class TickView:
    """One tick of a rollout, shaped like a StepOutput on the host."""

    def __init__(self, out, t):
        self.obs = out.obs[t].cpu().numpy()
        self.rewards = out.rewards[t].cpu().numpy()
        self.dones = out.dones[t].cpu().numpy()
        self.events = {k: v[t].cpu().numpy() for k, v in out.events.items()}
        inf = out.info
        self.info = {"alive": inf["alive"][t].cpu().numpy(), "alive_pre": inf["alive_pre"][t].cpu().numpy(),
                     "reason": inf["reason"][t].cpu().numpy(), "ttc_min": inf["ttc_min"][t].cpu().numpy(),
                     "state": {k: v[t].cpu().numpy() for k, v in inf["state"].items()},
                     "reward_terms": {k: v[t].cpu().numpy() for k, v in inf["reward_terms"].items()}}


def assert_same_engine(a: Engine, b: Engine):
    assert torch.equal(a.state_tensor, b.state_tensor)
    for k in ("alive", "reason", "event_seen", "spawn_step", "step_count"):
        assert torch.equal(a.device_tables()[k], b.device_tables()[k]), k


def assert_slot_equals_step(rb, slot, sb):
    assert torch.equal(rb.obs[slot], sb.obs)
    for k in OUT_VIEWS:
        assert torch.equal(rb.views[k][slot], sb.views[k]), k


@pytest.mark.parametrize("autoreset", [False, True])
@pytest.mark.parametrize("shape", [None, (4, 4), (16, 1), (4, 0, 1), (8, 0, 0), (7, 0, 2), (3, 0, 2), (1, 0, 2)])
def test_replayed_rollout_equals_steps(autoreset, shape, device):
    W, M, T = 8, 16, 48
    inp = C.build_inputs(cfg_of(W, M, seed=31))
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    if shape:
        a.tune(*shape)
        b.tune(*shape)
    acts = torch.from_numpy(event_actions(T, W, M)).to(device)
    ca = torch.zeros((W, 5), dtype=torch.int32, device=device)
    cb = torch.zeros_like(ca)
    rb = a.new_rollout_buffers(T)
    a.launch_step(acts, rb, autoreset=autoreset, ticks=T, event_counts=ca)
    sb = b.new_step_buffers()
    dones = 0
    for t in range(T):
        b.launch_step(acts[t], sb, autoreset=autoreset, event_counts=cb)
        assert_slot_equals_step(rb, t, sb)
        dones += int(sb.views["dones"].sum())
    assert_same_engine(a, b)
    assert torch.equal(ca, cb)
    assert a.step_count == b.step_count == T
    assert dones > 0


@pytest.mark.parametrize("W", [16, 1200])
def test_lane_follower_rollout_equals_fused_policy_steps(W, device):
    """Ticks >= 1 take the fused LaneFollower's actions from shared memory;
    the step-by-step reference ping-pongs them through next_actions."""
    M, T = 16, 24
    inp = C.build_inputs(cfg_of(W, M, seed=9))
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    a0 = torch.empty((W, M, 3), dtype=torch.float64, device=device)
    b.observe(as_numpy=False, next_actions=a0)
    out = a.rollout(a0.clone(), ticks=T, policy="lane_follower", autoreset=True)
    acts = [a0, torch.empty_like(a0)]
    sb = b.new_step_buffers()
    for t in range(T):
        b.launch_step(acts[t % 2], sb, autoreset=True, next_actions=acts[(t + 1) % 2])
        assert torch.equal(out.obs[t], sb.obs)
        for k in OUT_VIEWS:
            assert torch.equal(out._info_src[k][t], sb.views[k]), (t, k)
    assert torch.equal(out.next_actions, acts[T % 2])
    assert_same_engine(a, b)


def test_ring_slots_wrap(device):
    W, M, T, S, start = 4, 16, 7, 3, 1
    inp = C.build_inputs(cfg_of(W, M, seed=5))
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    acts = torch.from_numpy(philox_actions(4, T, W, M).astype(np.float64)).to(device)
    rb = a.new_rollout_buffers(S)
    a.launch_step(acts, rb, ticks=T, ring_start=start)
    steps = []
    for t in range(T):
        sb = b.new_step_buffers()
        b.launch_step(acts[t], sb)
        steps.append(sb)
    for t in range(T - S, T):
        assert_slot_equals_step(rb, (start + t) % S, steps[t])
    assert_same_engine(a, b)


@pytest.mark.parametrize("name", ["traj_c1", "traj_events", "traj_wet", "traj_bicycle", "traj_sparse",
                                  "traj_events_inv"])
def test_rollout_matches_oracle(name, device):
    case = case_inputs(name)
    gpu = Engine(**case.inputs.as_kwargs(), device=device)
    ora = OracleEngine(**case.inputs.as_kwargs())
    acts = case.actions[:case.steps].astype(np.float64)
    out = gpu.rollout(acts)
    dev = Dev()
    for t in range(case.steps):
        compare(dev, t + 1, TickView(out, t), ora.step(acts[t]), ora.obs_config)
    for k in EVENT_TYPES:
        assert np.array_equal(gpu.event_seen[k], ora.event_seen[k])
    assert gpu.step_count == case.steps


def test_rollout_rejects_nonfinite_before_running(device):
    inp = C.build_inputs(cfg_of(2, 4, assignment="fixed"))
    eng = Engine(**inp.as_kwargs(), device=device)
    before = eng.state_tensor.clone()
    acts = np.zeros((5, 2, 4, 3))
    acts[3, 1, 2, 1] = np.inf
    with pytest.raises(ValueError, match="world 1 agent 2"):
        eng.rollout(acts)
    assert torch.equal(before, eng.state_tensor)
    with pytest.raises(ValueError, match="shape"):
        eng.rollout(np.zeros((5, 2, 3, 3)))


def test_device_guard_stops_world_at_bad_tick(device):
    """Without the host check, the kernel stops a world at the tick whose
    actions are non-finite: that world holds its state after the previous
    ticks (what the step calls before the raising one would leave), the
    other worlds run the whole rollout."""
    W, M, T, bad_t = 3, 4, 6, 3
    inp = C.build_inputs(cfg_of(W, M, assignment="fixed"))
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    acts = torch.from_numpy(philox_actions(8, T, W, M).astype(np.float64)).to(device)
    acts[bad_t, 1, 2, 0] = float("nan")
    a.launch_step(acts, a.new_rollout_buffers(T), ticks=T)
    with pytest.raises(ValueError, match="world 1 agent 2"):
        a.raise_pending_error()
    sb = b.new_step_buffers()
    for t in range(T):
        x = acts[t].clone()
        if t >= bad_t:
            x[1] = 0.0
        b.launch_step(x, sb)
        if t == bad_t - 1:
            held = b.state_tensor[:, 1].clone()
    assert torch.equal(a.state_tensor[:, 1], held)
    assert torch.equal(a.state_tensor[:, 0], b.state_tensor[:, 0])
    assert torch.equal(a.state_tensor[:, 2], b.state_tensor[:, 2])
    assert int(a.device_tables()["step_count"][1]) == bad_t
    assert int(a.device_tables()["step_count"][0]) == T
