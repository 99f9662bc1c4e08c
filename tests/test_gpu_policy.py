"""Policy MLP on tcgen05 (BASELINE configs[4]) against its torch restatement
(oracle/policy.py) on the same weights.  The reference has no policy code, so
this parity is unpinned against the reference; the bar here:

* vs the bf16-emulating restatement (same rounding points as the kernel):
  |diff| <= 1e-4 + 1e-2 * |want|   (accumulation order, ex2.approx, bf16 rounding flips)
* vs plain float32: |diff| <= 3e-2 + 5e-2 * |want|   (bf16 operands)
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from cases import cfg_of
from oracle.policy import policy_forward
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.engine import Engine
from paper_2605_08528_b200.params import ObsConfig
from paper_2605_08528_b200.policy import PolicyMLP

pytestmark = pytest.mark.gpu


def env_obs(device, W=32, M=16, ticks=12, obs_config=None, seed=42):
    cfg = cfg_of(W, M, seed=seed)
    if obs_config is not None:
        cfg.obs = obs_config
    eng = Engine(**C.build_inputs(cfg).as_kwargs(), device=device)
    acts = torch.zeros((W, M, 3), dtype=torch.float64, device=device)
    obs = eng.observe(as_numpy=False, next_actions=acts)
    for _ in range(ticks):
        out = eng.step(acts.clone())
        obs = out.obs
        eng.lane_follower(obs, out=acts)
    return eng, obs.reshape(-1, obs.shape[-1]).contiguous()


def check(got, want, atol, rtol, what):
    got, want = got.double().cpu(), want.double().cpu()
    err = (got - want).abs()
    bound = atol + rtol * want.abs()
    worst = float((err - bound).max())
    print(f"{what}: max |diff| {float(err.max()):.3e}, max |want| {float(want.abs().max()):.3e}")
    assert worst <= 0, f"{what}: max |diff| {float(err.max())}"


@pytest.mark.parametrize("critic", [True, False])
def test_policy_forward_matches_torch(critic, device):
    eng, obs = env_obs(device)
    oc = eng.obs_config
    pol = PolicyMLP(oc, seed=3, device=device, critic=critic, head_scale=1.0)
    mean = torch.empty((obs.shape[0], 3), dtype=torch.float32, device=device)
    acts = torch.empty((obs.shape[0], 3), dtype=torch.float64, device=device)
    value = torch.empty((obs.shape[0],), dtype=torch.float32, device=device) if critic else None
    pol.forward(obs, actions=acts, mean=mean, value=value)
    torch.cuda.synchronize()
    sd = pol.state_dict()
    args = (sd, oc.ego_dim, oc.k_road, oc.k_vehicles)
    want16 = policy_forward(obs, *args, net="actor", bf16=True)
    want32 = policy_forward(obs, *args, net="actor", bf16=False)
    check(mean, want16, 1e-4, 1e-2, "actor vs bf16-emulated")
    check(mean, want32, 3e-2, 5e-2, "actor vs fp32")
    assert torch.equal(acts, mean.double())
    if critic:
        check(value, policy_forward(obs, *args, net="critic", bf16=True)[:, 0], 1e-4, 1e-2, "critic vs bf16")
        check(value, policy_forward(obs, *args, net="critic", bf16=False)[:, 0], 3e-2, 5e-2, "critic vs fp32")


def test_policy_ragged_and_empty_pools(device):
    """Row counts off the CTA tiles, agents without road points or neighbours,
    a reduced observation layout (k_road 20, k_vehicles 3, no weather)."""
    oc = ObsConfig(include_weather=False, k_road=20, k_vehicles=3, road_radius=12.5)
    eng, obs = env_obs(device, W=7, M=5, obs_config=oc, seed=19)
    obs = obs.clone()
    obs[3, oc.ego_dim:] = 0.0                                # no road, no neighbours
    obs[10, oc.ego_dim:oc.ego_dim + 5 * oc.k_road] = 0.0     # no road
    obs[11, oc.ego_dim + 5 * oc.k_road:] = 0.0               # no neighbours
    pol = PolicyMLP(oc, seed=5, device=device, head_scale=1.0)
    mean, value = pol(obs)
    torch.cuda.synchronize()
    sd = pol.state_dict()
    args = (sd, oc.ego_dim, oc.k_road, oc.k_vehicles)
    check(mean, policy_forward(obs, *args, net="actor", bf16=True), 1e-4, 1e-2, "actor")
    check(value, policy_forward(obs, *args, net="critic", bf16=True)[:, 0], 1e-4, 1e-2, "critic")


def test_policy_large_batch(device):
    """1024 x 16 agents (configs[4] size): every CTA of both kernels."""
    _, obs = env_obs(device, W=1024, M=16, ticks=4)
    pol = PolicyMLP(seed=9, device=device, head_scale=1.0)
    mean, value = pol(obs)
    torch.cuda.synchronize()
    sd = pol.state_dict()
    idx = torch.arange(0, obs.shape[0], 37, device=device)
    sub = obs[idx]
    check(mean[idx], policy_forward(sub, sd, 11, 350, 24, net="actor", bf16=True), 1e-4, 1e-2, "actor")
    check(value[idx], policy_forward(sub, sd, 11, 350, 24, net="critic", bf16=True)[:, 0], 1e-4, 1e-2, "critic")


@pytest.mark.parametrize("autoreset", [False, True])
def test_mlp_rollout_equals_step_loop(autoreset, device):
    """Engine.rollout(policy=PolicyMLP): T x (step launch -> policy forward)
    on the device equals the host-driven loop step -> policy -> step, bit for bit."""
    W, M, T = 8, 16, 40
    inp = C.build_inputs(cfg_of(W, M, seed=11))
    pol = PolicyMLP(seed=2, device=device, head_scale=1.0)
    a = torch.zeros((W, M, 3), dtype=torch.float64, device=device)
    a[..., 0] = 0.6
    ea = Engine(**inp.as_kwargs(), device=device)
    values = torch.empty((T, W, M), dtype=torch.float32, device=device)
    out = ea.rollout(a, ticks=T, autoreset=autoreset, policy=pol, values=values)
    torch.cuda.synchronize()
    eb = Engine(**inp.as_kwargs(), device=device)
    acts = a.clone()
    for t in range(T):
        o = eb.step(acts, autoreset=autoreset)
        mean, val = pol(o.obs)
        assert torch.equal(out.obs[t], o.obs), t
        assert torch.equal(out.rewards[t], o.rewards), t
        assert torch.equal(out.dones[t], o.dones), t
        assert torch.equal(values[t], val), t
        acts = mean.double()
    assert torch.equal(out.next_actions, acts)
    for k, v in ea.state.items():
        assert np.array_equal(v, eb.state[k]), k


def test_mlp_driven_env_matches_oracle(device):
    """The env under policy-MLP actions (the configs[4] loop) stays bit-exact
    against the CPU oracle on events / dones and within 1e-9 on state."""
    from oracle import OracleEngine
    from paper_2605_08528_b200.params import EVENT_TYPES, STATE_FIELDS
    W, M, T = 16, 16, 30
    inp = C.build_inputs(cfg_of(W, M, seed=13))
    gpu = Engine(**inp.as_kwargs(), device=device)
    ora = OracleEngine(**inp.as_kwargs())
    pol = PolicyMLP(seed=4, device=device, head_scale=1.0)
    acts = np.zeros((W, M, 3))
    acts[..., 0] = 0.8
    for t in range(T):
        g, o = gpu.step(acts), ora.step(acts)
        assert np.array_equal(g.dones, o.dones), t
        for k in EVENT_TYPES:
            assert np.array_equal(g.events[k], o.events[k]), (t, k)
        np.testing.assert_allclose(g.obs, o.obs, rtol=1e-6, atol=1e-6)
        mean, _ = pol(torch.as_tensor(g.obs, device=device))
        acts = mean.double().cpu().numpy()
    for k in STATE_FIELDS:
        np.testing.assert_allclose(gpu.state[k], ora.state[k], rtol=1e-9, atol=1e-9)


def test_ppo_sampling_matches_philox_restatement(device):
    """sample=True: actions = mean + exp(log_std) * eps with eps from the
    oracle's own Philox4x32-10 + Box-Muller; log-probabilities; statistics."""
    from oracle.policy import gaussian3
    _, obs = env_obs(device, W=64, M=16, ticks=4)
    pol = PolicyMLP(seed=6, device=device, head_scale=1.0)
    pol.log_std = torch.tensor([-0.5, 0.0, 0.3])
    n = obs.shape[0]
    mean = torch.empty((n, 3), dtype=torch.float32, device=device)
    acts = torch.empty((n, 3), dtype=torch.float64, device=device)
    a32 = torch.empty((n, 3), dtype=torch.float32, device=device)
    lp = torch.empty((n,), dtype=torch.float32, device=device)
    seed, ctr = 0x1234_5678_9ABC, 77
    pol.forward(obs, actions=acts, mean=mean, sample=True, seed=seed, counter=ctr, log_prob=lp, actions_f32=a32)
    torch.cuda.synchronize()
    z = gaussian3(n, seed, ctr)
    ls = pol.log_std.double().numpy()
    want = mean.double().cpu().numpy() + np.exp(ls) * z
    np.testing.assert_allclose(acts.cpu().numpy(), want, rtol=1e-12, atol=1e-12)
    assert torch.equal(a32, acts.float())
    want_lp = (-0.5 * z * z - ls - 0.5 * np.log(2 * np.pi)).sum(1)
    np.testing.assert_allclose(lp.double().cpu().numpy(), want_lp, rtol=1e-6, atol=1e-5)
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1.0) < 0.05
    # a different counter draws afresh; the same counter reproduces
    acts2 = torch.empty_like(acts)
    pol.forward(obs, actions=acts2, sample=True, seed=seed, counter=ctr + 1)
    acts3 = torch.empty_like(acts)
    pol.forward(obs, actions=acts3, sample=True, seed=seed, counter=ctr)
    torch.cuda.synchronize()
    assert not torch.equal(acts2, acts) and torch.equal(acts3, acts)


def test_gae_matches_numpy(device):
    from oracle.policy import gae as gae_ref
    from paper_2605_08528_b200.policy import gae
    rng = np.random.default_rng(3)
    T, N = 33, 1000
    r = rng.normal(size=(T, N))
    d = rng.uniform(size=(T, N)) < 0.05
    v = rng.normal(size=(T + 1, N)).astype(np.float32)
    adv, ret = gae(torch.as_tensor(r, device=device), torch.as_tensor(d, device=device),
                   torch.as_tensor(v, device=device), 0.99, 0.98)
    wa, wr = gae_ref(r, d, v, 0.99, 0.98)
    np.testing.assert_allclose(adv.cpu().numpy(), wa, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(ret.cpu().numpy(), wr, rtol=1e-5, atol=1e-5)


def test_ppo_rollout_records_a_batch(device):
    """configs[4] as a PPO collection: T ticks with sampled actions, their
    log-probs and values recorded per tick, then GAE over the batch; the
    recorded actions replayed through step() reproduce the rollout."""
    from paper_2605_08528_b200.policy import gae
    W, M, T = 16, 16, 24
    inp = C.build_inputs(cfg_of(W, M, seed=21))
    pol = PolicyMLP(seed=8, device=device, head_scale=1.0)
    a0 = torch.zeros((W, M, 3), dtype=torch.float64, device=device)
    ea = Engine(**inp.as_kwargs(), device=device)
    vals = torch.empty((T, W, M), dtype=torch.float32, device=device)
    lps = torch.empty((T, W, M), dtype=torch.float32, device=device)
    acts = torch.empty((T, W, M, 3), dtype=torch.float32, device=device)
    out = ea.rollout(a0, ticks=T, policy=pol, values=vals, sample=True, seed=5, log_probs=lps, actions_out=acts,
                     autoreset=True)
    torch.cuda.synchronize()
    eb = Engine(**inp.as_kwargs(), device=device)
    a = a0.clone()
    for t in range(T):
        o = eb.step(a, autoreset=True)
        assert torch.equal(o.obs, out.obs[t]) and torch.equal(o.rewards, out.rewards[t]), t
        _, val = pol(o.obs)
        assert torch.equal(val, vals[t])
        a = torch.empty((W, M, 3), dtype=torch.float64, device=device)
        pol.forward(o.obs, actions=a, sample=True, seed=5, counter=t)
        assert torch.equal(a.float(), acts[t])
    adv, ret = gae(out.rewards[1:], out.dones[1:], vals, 0.99, 0.98)
    assert adv.shape == (T - 1, W, M) and bool(torch.isfinite(adv).all())
