"""Host delivery of the numpy step path (dg_to_host): the observation reaches
the numpy array through mapped pinned slabs that carry only each row's
non-zero road / vehicle prefix over PCIe.  The arrays must equal the device
observation BIT FOR BIT on every step -- including rows whose prefix shrank
since the slab last held them -- and every returned array must stay a fresh
object (engine.py:363-364, 397-406): a slab is reused only after the caller
dropped every array of the step that filled it."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from cases import cfg_of, philox_actions
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.engine import Engine

pytestmark = pytest.mark.gpu


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("W,M,keep_every", [(8, 16, 3), (256, 16, 5), (3, 4, 2)])
def test_numpy_obs_bit_identical_to_device(W, M, keep_every, device):
    inp = C.build_inputs(cfg_of(W, M, seed=11))
    a = Engine(**inp.as_kwargs(), device=device)      # numpy path (mapped slabs)
    b = Engine(**inp.as_kwargs(), device=device)      # device path
    acts = philox_actions(77, 40, W, M).astype(np.float64)
    held = []
    for t in range(40):
        ga = a.step(acts[t], autoreset=True)
        gb = b.step(torch.from_numpy(acts[t]).to(device), autoreset=True)
        want = gb.obs.cpu().numpy()
        assert np.array_equal(bits(ga.obs), bits(want)), f"tick {t}: obs bits"
        assert np.array_equal(ga.rewards, gb.rewards.cpu().numpy()), f"tick {t}: rewards"
        assert np.array_equal(ga.dones, gb.dones.cpu().numpy()), f"tick {t}: dones"
        if t % keep_every == 0:
            held.append((ga, want.copy()))             # keeps its slab out of the pool
    for ga, want in held:                              # nothing later overwrote a held array
        assert np.array_equal(bits(ga.obs), bits(want))
    assert a._mapped_pool.slabs <= a._mapped_pool.max_slabs


def test_pool_exhaustion_falls_back_to_full_copy(device):
    W, M = 4, 16
    inp = C.build_inputs(cfg_of(W, M, seed=2))
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    a._mapped_pool.max_slabs = 2
    acts = philox_actions(5, 6, W, M).astype(np.float64)
    outs = []
    for t in range(6):
        outs.append(a.step(acts[t]))                   # every output held: slabs run out after 2
        want = b.step(torch.from_numpy(acts[t]).to(device)).obs.cpu().numpy()
        assert np.array_equal(bits(outs[-1].obs), bits(want))
    assert a._mapped_pool.slabs == 2


def test_shrinking_prefixes_are_zeroed(device):
    """A tick with long road prefixes followed, in the SAME slab, by a tick
    after every agent was teleported far off the road (empty road prefixes):
    the stale tails must read as zeros."""
    W, M = 4, 16
    inp = C.build_inputs(cfg_of(W, M, seed=3))
    a = Engine(**inp.as_kwargs(), device=device)
    b = Engine(**inp.as_kwargs(), device=device)
    z = np.zeros((W, M, 3))
    o1 = a.step(z)
    b.step(torch.zeros((W, M, 3), dtype=torch.float64, device=device))
    assert (o1.obs[..., 11:1761] != 0).sum() > 0
    del o1                                             # the slab goes back to the pool
    far = np.full((W, M, 2), 5000.0) + np.arange(W * M, dtype=np.float64).reshape(W, M, 1) * 50.0
    for e in (a, b):
        e.teleport_reset(np.ones((W, M), bool), new_starts=far)
    o2 = a.step(z)
    want = b.step(torch.zeros((W, M, 3), dtype=torch.float64, device=device)).obs.cpu().numpy()
    assert a._mapped_pool.slabs == 1                   # the same slab served both ticks
    assert np.array_equal(bits(o2.obs), bits(want))
    assert (o2.obs[..., 11:1761] != 0).sum() == 0


@pytest.mark.parametrize("mode", [2, 0, 1])
def test_prefix_record_bounds_the_nonzero_obs(mode, device):
    """DgStepIO.prefix_out (5 n_r, 7 n_v floats) equals the kernel's own
    candidate / neighbour counts and nothing past it is non-zero -- the
    property dg_to_host relies on -- in every launch mode."""
    W, M = 16, 16
    inp = C.build_inputs(cfg_of(W, M, seed=8))
    eng = Engine(**inp.as_kwargs(), device=device, launch_mode=mode)
    oc = eng.obs_config
    road0, veh0 = oc.ego_dim, oc.ego_dim + 5 * oc.k_road
    bufs = eng.new_step_buffers()
    ix = eng.new_index_buffer(1)
    px = torch.full((W, M, 2), -1, dtype=torch.int16, device=device)
    acts = philox_actions(9, 12, W, M).astype(np.float64)
    for t in range(12):
        eng.launch_step(torch.from_numpy(acts[t]).to(device), bufs, index_out=ix, prefix_out=px)
        p, i, o = px.cpu().numpy(), ix[0].cpu().numpy(), bufs.obs.cpu().numpy()
        assert np.array_equal(p[..., 0], 5 * i[..., 1]) and np.array_equal(p[..., 1], 7 * i[..., 2])
        cols = np.arange(o.shape[-1])
        past = ((cols >= road0) & (cols < veh0) & (cols >= road0 + p[..., :1])) | (cols >= veh0 + p[..., 1:])
        assert not np.any(o.view(np.uint32)[past]), f"tick {t}: non-zero obs past the prefix"
