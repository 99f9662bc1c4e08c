"""Episode safety metrics (SR, CR, DRAC) on the GPU.

Drop-in for ``drivegrid.metrics`` (``/root/reference/pkg/src/drivegrid/metrics.py``):

* ``pairwise_drac(pos, yaw, vel_world, r_hull, d_hull, alive)`` -- metrics.py:33-62,
  one launch of ``dg_pairwise_drac``;
* ``episode_metrics(log, valid, length, width, wheelbase, threshold)`` --
  metrics.py:86-125 over a recorded episode (``Engine.run_episode(record=True)``):
  every logged state goes to the device in one batch and one launch reduces the
  per-agent max over the steps;
* ``Engine.track_episode_metrics()`` / ``Engine.episode_metrics()`` -- the same
  numbers accumulated INSIDE the fused step kernel (running per-agent max DRAC
  on each tick's post-physics state over the agents alive before it, goal /
  collision latches), so a rollout needs no log at all.

``EpisodeMetrics`` has the reference's fields and ``to_dict``.  Across GPUs the
per-rank ``metric_summary`` (counts and the DRAC-over-threshold sum) is
all-gathered and combined in rank order (sharding.py).
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .tables import circle_layout

DRAC_THRESHOLD = 3.4  # m/s^2 (metrics.py:21)


@dataclass(frozen=True)
class EpisodeMetrics:
    sr: float
    cr: float
    mean_max_drac: float
    valid_agents: int
    goals: int
    collisions: int
    per_agent_max_drac: np.ndarray

    def to_dict(self) -> dict:
        return {"sr": self.sr, "cr": self.cr, "mean_max_drac": self.mean_max_drac,
                "valid_agents": self.valid_agents, "goals": self.goals, "collisions": self.collisions}


def drac(v_rel_closing: float, gap: float) -> float:
    """Scalar DRAC (metrics.py:24-30): v^2 / (2 d) when closing."""
    if gap <= 0:
        raise ValueError("gap must be positive")
    if v_rel_closing <= 0:
        return 0.0
    return v_rel_closing ** 2 / (2.0 * gap)


def _dev(a, dtype, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a)).to(device=device, dtype=dtype)


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("drivegrid-b200 metrics need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _launch(x, y, yaw, vx, vy, alive, r_hull, d_hull, out, accumulate: bool, world_velocity: bool):
    lib = N.load_library()
    steps, W, M = x.shape
    stream = ct.c_void_p(torch.cuda.current_stream(out.device).cuda_stream)
    N.check(lib, lib.dg_pairwise_drac(x.data_ptr(), y.data_ptr(), yaw.data_ptr(), vx.data_ptr(),
                                      vy.data_ptr(), alive.data_ptr(), r_hull.data_ptr(),
                                      d_hull.data_ptr(), steps, W, M, out.data_ptr(),
                                      int(accumulate), int(world_velocity), stream),
            "dg_pairwise_drac")


def pairwise_drac(pos, yaw, vel_world, r_hull, d_hull, alive, as_numpy: bool = True):
    """Per-agent max DRAC against alive neighbours for one state snapshot
    (metrics.py:33-62).  pos / vel_world (W, M, 2), yaw / r_hull / d_hull /
    alive (W, M)."""
    dev = _device()
    pos = _dev(pos, torch.float64, dev)
    vel = _dev(vel_world, torch.float64, dev)
    yaw = _dev(yaw, torch.float64, dev)
    W, M = yaw.shape
    out = torch.zeros((W, M), dtype=torch.float64, device=dev)
    one = lambda t: t.contiguous().reshape(1, W, M)  # noqa: E731
    _launch(one(pos[..., 0]), one(pos[..., 1]), one(yaw), one(vel[..., 0]), one(vel[..., 1]),
            one(_dev(alive, torch.uint8, dev)), _dev(r_hull, torch.float64, dev),
            _dev(d_hull, torch.float64, dev), out, accumulate=False, world_velocity=True)
    return out.cpu().numpy() if as_numpy else out


def _records(log):
    return log.steps if hasattr(log, "steps") else log


def episode_metrics(log, valid: np.ndarray, length=None, width=None, wheelbase: float = 2.6,
                    threshold: float = DRAC_THRESHOLD) -> EpisodeMetrics:
    """Aggregate a recorded episode into SR / CR / mean peak DRAC
    (metrics.py:86-125): SR and CR over valid spawns whose goal / collision
    event fired at least once; DRAC averages the per-agent episode maxima that
    exceed ``threshold``."""
    valid = np.asarray(valid, dtype=bool)
    W, M = valid.shape
    length = length if length is not None else np.full((W, M), 4.0)
    width = width if width is not None else np.full((W, M), 2.0)
    r_hull, d_hull = circle_layout(np.asarray(length, np.float64), np.asarray(width, np.float64), wheelbase)
    recs = _records(log)
    goal_seen = np.zeros((W, M), dtype=bool)
    coll_seen = np.zeros((W, M), dtype=bool)
    for rec in recs:
        goal_seen |= np.asarray(rec["events"]["goal"], dtype=bool)
        coll_seen |= np.asarray(rec["events"]["collision"], dtype=bool)
    dev = _device()
    max_drac = torch.zeros((W, M), dtype=torch.float64, device=dev)
    if recs:
        def stack(key, dtype, src="state"):
            cols = [rec[src][key] if src else rec[key] for rec in recs]
            if isinstance(cols[0], torch.Tensor):
                return torch.stack([c.to(dev) for c in cols]).to(dtype).contiguous()
            return _dev(np.stack([np.asarray(c) for c in cols]), dtype, dev)

        _launch(stack("x", torch.float64), stack("y", torch.float64), stack("yaw", torch.float64),
                stack("v_x", torch.float64), stack("v_y", torch.float64),
                stack("alive_pre", torch.uint8, src=None), _dev(r_hull, torch.float64, dev),
                _dev(d_hull, torch.float64, dev), max_drac, accumulate=False, world_velocity=False)
    return aggregate(goal_seen, coll_seen, max_drac.cpu().numpy(), valid, threshold)


def aggregate(goal_seen, coll_seen, max_drac, valid, threshold: float = DRAC_THRESHOLD) -> EpisodeMetrics:
    """metrics.py:110-125 on per-agent latches and maxima."""
    valid = np.asarray(valid, dtype=bool)
    n_valid = int(valid.sum())
    goals = int((np.asarray(goal_seen, bool) & valid).sum())
    colls = int((np.asarray(coll_seen, bool) & valid).sum())
    over = max_drac[valid & (max_drac > threshold)]
    return EpisodeMetrics(
        sr=goals / n_valid if n_valid else 0.0,
        cr=colls / n_valid if n_valid else 0.0,
        mean_max_drac=float(over.mean()) if over.size else 0.0,
        valid_agents=n_valid, goals=goals, collisions=colls, per_agent_max_drac=max_drac)


# the CASPS harness (metrics.py:130-250 of the reference) lives in casps.py
from .casps import BenchReport, measure_engine, run_bench, write_bench_csv  # noqa: E402,F401
