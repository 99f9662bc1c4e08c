"""Host side of the policy MLP (no GPU): the canonical UMMA tile packing,
the folded first layer, the torch restatement's two modes agreeing."""

from __future__ import annotations

import numpy as np
import torch

from oracle.policy import policy_forward
from paper_2605_08528_b200.policy import LN2, LOG2E, PolicyMLP, fold_first_layer, kmajor_tile


def test_kmajor_tile_positions():
    w = np.arange(16 * 32, dtype=np.float32).reshape(16, 32) / 64.0   # exact in bf16
    t = kmajor_tile(w, 32).view(np.uint16)
    bf = lambda x: int(torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).view(torch.int16)) & 0xFFFF  # noqa: E731
    for r, k in ((0, 0), (1, 0), (7, 7), (0, 8), (8, 0), (9, 17), (15, 31)):
        off = ((r // 8) * (32 // 8) + k // 8) * 128 + (r % 8) * 16 + (k % 8) * 2
        assert t[off // 2] == bf(w[r, k]), (r, k)


def test_fold_first_layer_is_exact_algebra():
    rng = np.random.default_rng(0)
    w, b = rng.normal(size=(96, 5)), rng.normal(size=96)
    x = rng.normal(size=(10, 5))
    f = fold_first_layer(w, b).astype(np.float64)
    y = np.concatenate([x, np.ones((10, 1))], axis=1) @ f.T
    np.testing.assert_allclose(y / LOG2E, x @ w.T + b, rtol=1e-6, atol=1e-6)
    assert abs(LOG2E * LN2 - 1.0) < 1e-15


def test_torch_restatement_modes_agree():
    pol = PolicyMLP(device="cpu", seed=1, head_scale=1.0)
    sd = pol.state_dict()
    g = torch.Generator().manual_seed(0)
    A, k_road, k_veh = 64, 350, 24
    obs = torch.zeros((A, 11 + 5 * k_road + 7 * k_veh))
    obs[:, :11] = torch.rand((A, 11), generator=g) * 2 - 1
    for a in range(A):
        nr, nv = a % 40, a % 16                           # includes agents with empty pools
        road = obs[a, 11:11 + 5 * k_road].view(k_road, 5)
        road[:nr] = torch.rand((nr, 5), generator=g) * 2 - 1
        road[:nr, 3] = 0.6
        veh = obs[a, 11 + 5 * k_road:].view(k_veh, 7)
        veh[:nv] = torch.rand((nv, 7), generator=g) * 2 - 1
        veh[:nv, 2] = 0.04
    for net in ("actor", "critic"):
        a32 = policy_forward(obs, sd, 11, k_road, k_veh, net=net, bf16=False)
        a16 = policy_forward(obs, sd, 11, k_road, k_veh, net=net, bf16=True)
        assert torch.isfinite(a32).all()
        np.testing.assert_allclose(a16.numpy(), a32.numpy(), rtol=5e-2, atol=3e-2)


def test_state_dict_round_trip():
    a = PolicyMLP(device="cpu", seed=1)
    b = PolicyMLP(device="cpu", seed=2)
    b.load_state_dict(a.state_dict())
    for k, v in a.state_dict().items():
        assert torch.equal(v, b.state_dict()[k]), k
