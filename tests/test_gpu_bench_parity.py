"""Parity on the exact configurations bench.py times.

* 256 x 16 default pool (seed 42), 200 ticks of a float32 Philox action
  stream, one fused launch per tick (the Engine.step path);
* 256 x 16, the bench path itself: persistent 64-tick launches with the
  LaneFollower and the autoreset fused into the step, outputs written to a
  wrapping rollout ring -- against OracleEngine.step + teleport_reset(dones)
  driven by the LaneFollower on the ORACLE's observations, 256 ticks;
* 512 x 16, the C4/C5 kernel variant (world_step_kernel<1, 128, 4>: 4 warps
  per world, 4 CTAs per SM, spatial index on) in both modes.

Every tick: dones / events / reason / alive / alive_pre bit-exact, the integer
decisions behind the floats -- nearest-lane index (rewards.py:94 argmin),
road slot -> segment map (observation.py:96-99 stable argsort) and neighbour
order (observation.py:246 stable argsort) -- compared AS INTEGERS through the
kernel's ``index_out`` record; floats within 1e-9 (f64) / 1e-6 (f32 obs).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from cases import philox_actions
from oracle import OracleEngine
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.engine import Engine
from paper_2605_08528_b200.params import EVENT_TYPES, STATE_FIELDS
from paper_2605_08528_b200.policies import LaneFollower
from test_gpu_parity import OBS_ATOL, OBS_RTOL, Dev

pytestmark = pytest.mark.gpu

TERMS = ("progress", "lane", "offroad", "idle", "ttc_vehicle", "ttc_edge", "total")


def headline_inputs(W=256, M=16):
    cfg = C.RootConfig()
    cfg.env.num_envs, cfg.env.num_agents_per_env = W, M
    return C.build_inputs(cfg)


def compare_indices(t, ix: np.ndarray, rec, take_veh: int):
    """ix: [W][M][stride] int32 record of one tick; rec: oracle IndexRecord."""
    ctx = f"tick {t}"
    assert np.array_equal(ix[..., 0], rec.lane), f"{ctx}: nearest-lane index"
    assert np.array_equal(ix[..., 1], rec.road_n), f"{ctx}: road candidates kept"
    assert np.array_equal(ix[..., 2], rec.veh_n), f"{ctx}: valid neighbours"
    veh = ix[..., 3:3 + take_veh]
    keep = np.arange(take_veh) < rec.veh_n[..., None]
    assert np.array_equal(np.where(keep, veh, -1), np.where(keep, rec.veh, -1)), f"{ctx}: neighbour order"
    road = ix[..., 3 + take_veh:]
    assert road.shape == rec.road.shape
    keep = np.arange(road.shape[-1]) < rec.road_n[..., None]
    assert np.array_equal(np.where(keep, road, -1), np.where(keep, rec.road, -1)), f"{ctx}: road slot map"


def compare_tick(dev: Dev, t, views: dict, slot: int, obs: np.ndarray, ix: np.ndarray, o, take_veh: int):
    """One tick of device ring outputs (``views`` of new_rollout_buffers at
    ``slot``) against one OracleEngine.step result ``o``."""
    ctx = f"tick {t}"
    v = {k: a[slot].cpu().numpy() for k, a in views.items()}
    assert np.array_equal(v["dones"].astype(bool), o.dones), f"{ctx} dones"
    ev = v["events"].astype(bool)
    for i, k in enumerate(EVENT_TYPES):
        assert np.array_equal(ev[..., i], o.events[k]), f"{ctx} event {k}"
    assert np.array_equal(v["reason"], o.info["reason"]), f"{ctx} reason"
    assert np.array_equal(v["alive"].astype(bool), o.info["alive"]), f"{ctx} alive"
    assert np.array_equal(v["alive_pre"].astype(bool), o.info["alive_pre"]), f"{ctx} alive_pre"
    compare_indices(t, ix, o.info["indices"], take_veh)
    dev.f("rewards", v["rewards"], o.rewards)
    dev.f("ttc_min", v["ttc_min"], o.info["ttc_min"])
    for i, k in enumerate(TERMS):
        dev.f(f"term_{k}", v["terms"][i], o.info["reward_terms"][k])
    for i, k in enumerate(STATE_FIELDS):
        dev.f(f"snap_{k}", v["snapshot"][i], o.info["state"][k])
    dev.f("obs", obs, o.obs, rtol=OBS_RTOL, atol=OBS_ATOL)


def run_philox(device, W, M, ticks, shape=None, launch_mode=None):
    inp = headline_inputs(W, M)
    gpu = Engine(**inp.as_kwargs(), device=device, launch_mode=launch_mode)
    if shape is not None:
        assert gpu.launch_shape() == shape
    ora = OracleEngine(**inp.as_kwargs(), num_workers=16)
    ora.record_indices = True
    take_veh = min(gpu.obs_config.k_vehicles, M)
    acts = philox_actions(2024, ticks, W, M)
    bufs = gpu.new_rollout_buffers(1)
    ix = gpu.new_index_buffer(1)
    dev = Dev()
    for t in range(ticks):
        a = acts[t].astype(np.float64)
        o = ora.step(a)
        gpu.launch_step(torch.from_numpy(a).to(device), bufs, index_out=ix)
        compare_tick(dev, t + 1, bufs.views, 0, bufs.obs[0].cpu().numpy(), ix[0].cpu().numpy(), o, take_veh)
    st = gpu.state
    for k in STATE_FIELDS:
        dev.f(f"state_{k}", st[k], ora.state[k])
    assert np.array_equal(gpu.alive, ora.alive) and np.array_equal(gpu.reason, ora.reason)
    return dev, ora


def run_bench_path(device, W, M, launches, R=64, ring=None, shape=None, launch_mode=None, inp=None,
                   autoreset=True):
    """bench.py's timed loop (persistent R-tick launches, fused LaneFollower +
    autoreset, ring_start = tick % ring) against the oracle driven the same
    way on its own observations."""
    inp = inp if inp is not None else headline_inputs(W, M)
    W, M = inp.sim.num_envs, inp.sim.num_agents
    gpu = Engine(**inp.as_kwargs(), device=device, launch_mode=launch_mode)
    if shape is not None:
        assert gpu.launch_shape() == shape
    ora = OracleEngine(**inp.as_kwargs(), num_workers=16)
    ora.record_indices = True
    pol = LaneFollower(obs_config=ora.obs_config)
    take_veh = min(gpu.obs_config.k_vehicles, M)
    ring = ring or R + 8                       # wraps from the second launch on
    rb = gpu.new_rollout_buffers(ring)
    ix = gpu.new_index_buffer(ring)
    acts = torch.zeros((W, M, 3), dtype=torch.float64, device=device)
    gobs0 = gpu.observe(out=rb.obs[ring - 1], as_numpy=False, next_actions=acts)
    obs = ora.observe()
    np.testing.assert_allclose(gobs0.cpu().numpy(), obs, rtol=OBS_RTOL, atol=OBS_ATOL)
    dev, tick, resets, act_mismatch = Dev(), 0, 0, 0
    for _ in range(launches):
        start = tick % ring
        gpu.launch_step(acts, rb, autoreset=autoreset, next_actions=acts, ticks=R, ring_start=start, index_out=ix)
        torch.cuda.synchronize()
        obs_ring = rb.obs  # [ring][W][M][D]
        for t in range(R):
            a = pol(obs)
            o = ora.step(a)
            if autoreset:
                ora.teleport_reset(o.dones)
            resets += int(o.dones.sum())
            slot = (start + t) % ring
            compare_tick(dev, tick + t + 1, rb.views, slot, obs_ring[slot].cpu().numpy(),
                         ix[slot].cpu().numpy(), o, take_veh)
            obs = o.obs
        tick += R
        # the fused policy's actions for the next launch == the LaneFollower on the oracle's last obs
        want = pol(obs)
        got = acts.cpu().numpy()
        act_mismatch += int((got != want).sum())
        assert np.array_equal(got, want), "fused LaneFollower actions"
    st = gpu.state
    for k in STATE_FIELDS:
        dev.f(f"state_{k}", st[k], ora.state[k])
    assert np.array_equal(gpu.alive, ora.alive) and np.array_equal(gpu.reason, ora.reason)
    assert np.array_equal(gpu.spawn_step, ora.spawn_step)
    return dev, resets


HEADLINE_SHAPES = {2: {"mode": "fused+physics-warp", "warps": 7, "ctas_per_sm": 0},
                   0: {"mode": "fused", "warps": 8, "ctas_per_sm": 0}}


@pytest.mark.parametrize("mode", [2, 0])
def test_headline_philox_stream_200_ticks(mode, device):
    dev, ora = run_philox(device, 256, 16, 200, shape=HEADLINE_SHAPES[mode], launch_mode=mode)
    print("\n[256x16 philox, 200 ticks] max |gpu - oracle|:", {k: f"{v:.2e}" for k, v in sorted(dev.max.items())})


@pytest.mark.parametrize("mode", [2, 0])
def test_headline_bench_path_256_ticks(mode, device):
    dev, resets = run_bench_path(device, 256, 16, launches=4, shape=HEADLINE_SHAPES[mode], launch_mode=mode)
    assert resets > 0                        # the autoreset path ran
    print(f"\n[256x16 bench path, 4 x 64 ticks, {resets} resets] max |gpu - oracle|:",
          {k: f"{v:.2e}" for k, v in sorted(dev.max.items())})


@pytest.mark.parametrize("mode", [2, 0])
def test_timeout_and_park_in_persistent_launch(mode, device):
    """No autoreset, episode_len 25 (the traj_timeout fixture's config): in
    one 40-tick launch agents collide / leave the lane and are parked, the
    survivors time out at tick 25 and stay dead -- the physics warp's
    next-tick guess is wrong for every one of them and must be redone."""
    from cases import case_inputs
    inp = case_inputs("traj_timeout").inputs
    dev, finished = run_bench_path(device, 0, 0, launches=1, R=40, ring=40, launch_mode=mode, inp=inp,
                                   autoreset=False)
    assert finished > 0


def test_c4_variant_philox_64_ticks(device):
    dev, _ = run_philox(device, 512, 16, 64, shape={"mode": "fused", "warps": 4, "ctas_per_sm": 4})
    print("\n[512x16 philox] max |gpu - oracle|:", {k: f"{v:.2e}" for k, v in sorted(dev.max.items())})


def test_c4_variant_bench_path_64_ticks(device):
    dev, resets = run_bench_path(device, 512, 16, launches=1, ring=64,
                                 shape={"mode": "fused", "warps": 4, "ctas_per_sm": 4})
    print(f"\n[512x16 bench path, {resets} resets] max |gpu - oracle|:",
          {k: f"{v:.2e}" for k, v in sorted(dev.max.items())})


@pytest.mark.parametrize("mode", [0, 1])
def test_index_record_both_launch_modes(mode, device):
    """The index record is a debug output of both kernels (fused and split)."""
    inp = headline_inputs(8, 16)
    gpu = Engine(**inp.as_kwargs(), device=device, launch_mode=mode)
    ora = OracleEngine(**inp.as_kwargs())
    ora.record_indices = True
    acts = philox_actions(7, 30, 8, 16)
    bufs = gpu.new_rollout_buffers(1)
    ix = gpu.new_index_buffer(1)
    dev = Dev()
    for t in range(30):
        a = acts[t].astype(np.float64)
        o = ora.step(a)
        gpu.launch_step(torch.from_numpy(a).to(device), bufs, index_out=ix)
        compare_tick(dev, t + 1, bufs.views, 0, bufs.obs[0].cpu().numpy(), ix[0].cpu().numpy(), o, 16)
