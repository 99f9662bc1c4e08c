"""Torch restatement of the policy MLP -- TEST INFRASTRUCTURE ONLY.

The reference package has no policy code; the network is the paper's App. E
(PAPER.md:752-768).  Parity for the device forward is therefore UNPINNED
against the reference: this module is the spec the tests check the tcgen05
kernels against, on the same weights (``PolicyMLP.state_dict()``).

``bf16=False``: plain float32 (masked max-pool with -inf padding).
``bf16=True``: the same graph with the kernel's rounding points emulated --
bf16 weights and layer inputs, fp32 accumulation, pooling on the raw layer-2
output (rounded to bf16; rounding is monotone, so the max of rounded values is
the rounded max) before bias + ELU, with the encoders' first layer in the
kernel's folded form ([W1 | b1] * log2 e against [x, 1]; W2 * ln 2) -- for a
tight comparison.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

LOG2E = 1.4426950408889634
LN2 = 0.6931471805599453
LAYERS = ("ego1", "ego2", "road1", "road2", "veh1", "veh2", "t1", "t2")


def _bf(x):
    return x.to(torch.bfloat16).to(torch.float32)


def _lin(x, w, b, bf16):
    if bf16:
        return _bf(x) @ _bf(w).t() + b
    return x @ w.t() + b


def policy_forward(obs: torch.Tensor, sd: dict, ego_dim: int, k_road: int, k_veh: int, net: str = "actor",
                   bf16: bool = False) -> torch.Tensor:
    """obs [A, D] float32 -> actor mean [A, 3] or critic value [A, 1]."""
    obs = obs.float()
    A = obs.shape[0]
    p = {n: (sd[f"{net}.{n}.weight"].to(obs.device), sd[f"{net}.{n}.bias"].to(obs.device))
         for n in LAYERS + ("head",)}
    ego = obs[:, :ego_dim]
    road = obs[:, ego_dim:ego_dim + 5 * k_road].reshape(A, k_road, 5)
    veh = obs[:, ego_dim + 5 * k_road:].reshape(A, k_veh, 7)
    road_ok = (road[..., 3] != 0) | (road[..., 4] != 0)       # unit direction: never (0, 0) when valid
    veh_ok = veh[..., 2] != 0                                   # length / 100 > 0 when valid

    def enc(x, ok, l1, l2):
        if bf16:
            # the kernel's folded form (exact algebra, different rounding points):
            # y = [x, 1] . ([W1 | b1] * log2 e),  h' = log2 e * ELU(y / log2 e),
            # z = h' . (W2 * ln 2)
            w1, b1 = p[l1]
            wf = (torch.cat([w1.double(), b1.double()[:, None]], dim=1) * LOG2E).float()
            y = _bf(torch.cat([x, torch.ones_like(x[..., :1])], dim=-1)) @ _bf(wf).t()
            h = torch.where(y > 0, y, LOG2E * (torch.exp2(y) - 1.0))
            w2 = (p[l2][0].double() * LN2).float()
            z = _bf(_bf(h) @ _bf(w2).t())                       # raw layer-2 accumulator, bf16
            z = z.masked_fill(~ok[..., None], float("-inf")).amax(dim=1)
            out = F.elu(z + p[l2][1])
        else:
            h = F.elu(_lin(x, *p[l1], bf16))
            z = F.elu(h @ p[l2][0].t() + p[l2][1])
            out = z.masked_fill(~ok[..., None], float("-inf")).amax(dim=1)
        return torch.where(ok.any(dim=1, keepdim=True), out, torch.zeros_like(out))

    e = F.elu(_lin(F.elu(_lin(ego, *p["ego1"], bf16)), *p["ego2"], bf16))
    r = enc(road, road_ok, "road1", "road2")
    v = enc(veh, veh_ok, "veh1", "veh2")
    x = torch.cat([e, r, v], dim=-1)
    h = F.elu(_lin(F.elu(_lin(x, *p["t1"], bf16)), *p["t2"], bf16))
    return h @ p["head"][0].t() + p["head"][1]


# ---------------------------------------------------------------- PPO sampling / GAE
M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(counter: "np.ndarray", key: tuple) -> "np.ndarray":
    """Philox4x32-10 (Salmon et al. 2011) over rows of uint32 counters [n, 4]."""
    import numpy as np
    c = counter.astype(np.uint64)
    k0, k1 = np.uint64(key[0]), np.uint64(key[1])
    for _ in range(10):
        p0 = np.uint64(M0) * c[:, 0]
        p1 = np.uint64(M1) * c[:, 2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK)
        c = np.stack([hi1 ^ c[:, 1] ^ k0, lo1, hi0 ^ c[:, 3] ^ k1, lo0], axis=1)
        k0 = (k0 + np.uint64(W0)) & np.uint64(MASK)
        k1 = (k1 + np.uint64(W1)) & np.uint64(MASK)
    return c.astype(np.uint32)


def gaussian3(n: int, seed: int, counter: int) -> "np.ndarray":
    """The three standard normals the kernel draws for rows 0..n-1 (Box-Muller, float64)."""
    import numpy as np
    rows = np.arange(n, dtype=np.uint64)
    ctr = np.stack([rows & np.uint64(MASK), rows >> np.uint64(32),
                    np.full(n, counter & MASK, dtype=np.uint64), np.full(n, counter >> 32, dtype=np.uint64)], axis=1)
    u = (philox4x32_10(ctr, (seed & MASK, seed >> 32)).astype(np.float64) + 0.5) * 2.0 ** -32
    r0, r1 = np.sqrt(-2.0 * np.log(u[:, 0])), np.sqrt(-2.0 * np.log(u[:, 2]))
    return np.stack([r0 * np.cos(2.0 * np.pi * u[:, 1]), r0 * np.sin(2.0 * np.pi * u[:, 1]),
                     r1 * np.cos(2.0 * np.pi * u[:, 3])], axis=1)


def gae(rewards, dones, values, gamma=0.99, lam=0.98):
    """delta_t = r_t + g V_{t+1} (1 - d_t) - V_t;  A_t = delta_t + g l (1 - d_t) A_{t+1} (float64)."""
    import numpy as np
    T = rewards.shape[0]
    adv = np.zeros(rewards.shape)
    a = np.zeros(rewards.shape[1:])
    for t in range(T - 1, -1, -1):
        nt = 1.0 - dones[t].astype(np.float64)
        delta = rewards[t] + gamma * values[t + 1].astype(np.float64) * nt - values[t].astype(np.float64)
        a = delta + gamma * lam * nt * a
        adv[t] = a
    return adv, adv + values[:T].astype(np.float64)
