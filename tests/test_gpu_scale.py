"""Full-size checks (BASELINE configs[3]: 4096 worlds x 16 agents, sharded by
world across GPUs).  This run has one GPU, so the shards run as separate
engines on it: each shard of a globally built batch must reproduce the same
worlds of the unsharded 4096 x 16 engine bit for bit over a fused-policy
rollout (the property that makes the N-GPU run exact), and size-independent
invariants must hold at full size."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.engine import Engine
from paper_2605_08528_b200.params import EVENT_TYPES
from paper_2605_08528_b200.sharding import shard_inputs, shard_range

pytestmark = pytest.mark.gpu

W, M, T = 4096, 16, 24


def _rollout(eng, T, dev):
    acts = torch.zeros((eng.W, eng.M, 3), dtype=torch.float64, device=dev)
    eng.observe(as_numpy=False, next_actions=acts)
    counters = torch.zeros((eng.W, 5), dtype=torch.int32, device=dev)
    rb = eng.new_rollout_buffers(T)
    eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=T, event_counts=counters)
    torch.cuda.synchronize()
    return rb, counters


@pytest.mark.parametrize("n_shards", [2, 8])
def test_world_shards_reproduce_the_full_batch(n_shards, device):
    cfg = C.RootConfig()
    cfg.env.num_envs, cfg.env.num_agents_per_env = W, M
    inp = C.build_inputs(cfg)
    full = Engine(**inp.as_kwargs(), device=device)
    rb, cnt = _rollout(full, T, device)
    for r in range(n_shards):
        lo, hi = shard_range(W, r, n_shards)
        sh = Engine(**shard_inputs(inp, r, n_shards).as_kwargs(), device=device)
        srb, scnt = _rollout(sh, T, device)
        assert torch.equal(srb.obs, rb.obs[:, lo:hi]), r
        for k in ("rewards", "dones", "events", "reason", "alive", "ttc_min"):
            assert torch.equal(srb.views[k], rb.views[k][:, lo:hi]), (r, k)
        assert torch.equal(sh.state_tensor, full.state_tensor[:, lo:hi]), r
        assert torch.equal(scnt, cnt[lo:hi]), r
        del sh, srb


def test_full_size_invariants(device):
    """4096 x 16 fused-policy rollout: counters equal the per-tick event sums,
    one-hot events, dones imply an event or timeout, obs rows of finished
    agents were written, determinism across two engines."""
    cfg = C.RootConfig()
    cfg.env.num_envs, cfg.env.num_agents_per_env = W, M
    inp = C.build_inputs(cfg)
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    rba, ca = _rollout(a, T, device)
    rbb, cb = _rollout(b, T, device)
    assert torch.equal(rba.obs, rbb.obs) and torch.equal(ca, cb)
    ev = rba.views["events"].to(torch.int32)                  # [T][W][M][4]
    assert int(ev.sum(-1).max()) <= 1                          # one-hot
    per_world = ev.sum(dim=(0, 2))                            # [W][4]
    assert torch.equal(per_world, ca[:, :4])
    alive_pre = rba.views["alive_pre"].to(torch.int32).sum(dim=(0, 2))
    assert torch.equal(alive_pre, ca[:, 4])
    dones = rba.views["dones"].bool()
    assert bool((~dones | (ev.sum(-1) > 0)).all())             # no timeouts inside 24 ticks
    valid = torch.as_tensor(a.valid, device=device)
    assert bool((rba.views["alive_pre"].bool() <= valid[None]).all())
    assert int(ca[:, 4].sum()) == T * int(valid.sum())        # autoreset keeps every valid slot alive
