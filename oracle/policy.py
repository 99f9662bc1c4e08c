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
