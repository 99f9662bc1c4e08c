"""Policy MLP on tcgen05 (BASELINE configs[4]) against its torch restatement
(oracle/policy.py) on the same weights.  The reference has no policy code, so
this parity is unpinned against the reference; the bar here:

* vs the bf16-emulating restatement (same rounding points as the kernel):
  |diff| <= 1e-5 + 1e-3 * |want|   (fp32 accumulation order only; observed 6e-8)
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
    check(mean, want16, 1e-5, 1e-3, "actor vs bf16-emulated")
    check(mean, want32, 3e-2, 5e-2, "actor vs fp32")
    assert torch.equal(acts, mean.double())
    if critic:
        check(value, policy_forward(obs, *args, net="critic", bf16=True)[:, 0], 1e-5, 1e-3, "critic vs bf16")
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
    check(mean, policy_forward(obs, *args, net="actor", bf16=True), 1e-5, 1e-3, "actor")
    check(value, policy_forward(obs, *args, net="critic", bf16=True)[:, 0], 1e-5, 1e-3, "critic")


def test_policy_large_batch(device):
    """1024 x 16 agents (configs[4] size): every CTA of both kernels."""
    _, obs = env_obs(device, W=1024, M=16, ticks=4)
    pol = PolicyMLP(seed=9, device=device, head_scale=1.0)
    mean, value = pol(obs)
    torch.cuda.synchronize()
    sd = pol.state_dict()
    idx = torch.arange(0, obs.shape[0], 37, device=device)
    sub = obs[idx]
    check(mean[idx], policy_forward(sub, sd, 11, 350, 24, net="actor", bf16=True), 1e-5, 1e-3, "actor")
    check(value[idx], policy_forward(sub, sd, 11, 350, 24, net="critic", bf16=True)[:, 0], 1e-5, 1e-3, "critic")
