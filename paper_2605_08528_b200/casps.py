"""CASPS harness: ``measure_engine`` / ``run_bench`` / ``BenchReport`` /
``write_bench_csv`` (drivegrid metrics.py:130-250), re-exported
by ``metrics``.

Same report fields, CSV row layout and grid / repeat logic as the reference;
the paths differ because the engine does:

* ``"vectorized"`` -- the reference-facing API: ``Engine.step(numpy)`` with the
  numpy LaneFollower on the host (inputs up, the whole observation batch down,
  every tick);
* ``"device"`` -- the same closed loop with observations, actions and the
  LaneFollower kept in HBM (``observe_device`` + the ``lane_follower`` kernel +
  ``step(cuda tensor)``), i.e. what a GPU-resident policy sees.

The reference's third path (its scalar ``reference_step``) is CPU code with no
place in this package; ``bench.py --impl reference`` times the CPU restatement
instead.  CASPS counts agents alive before each tick, like the reference; the
wall clock is bracketed by device synchronisation.
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass, field

import torch

from .params import PHASES
from .policies import LaneFollower

PATHS = ("vectorized", "device")


@dataclass
class BenchReport:
    num_envs: int
    num_agents: int
    backend: str
    path: str
    casps: float
    steps: int
    warmup_steps: int
    wall_seconds: float
    phase_ms: dict = field(default_factory=dict)
    workers: int = 1

    def to_row(self) -> dict:
        row = {"W": self.num_envs, "M": self.num_agents, "backend": self.backend, "path": self.path,
               "CASPS": round(self.casps, 1), "steps": self.steps, "wall_s": round(self.wall_seconds, 4)}
        row.update({f"{k}_ms": round(self.phase_ms.get(k, 0.0), 3) for k in PHASES})
        return row


def _host_loop(engine, policy, n: int):
    obs, ticks = engine.observe(), 0
    for _ in range(n):
        ticks += int(engine.alive.sum())
        obs = engine.step(policy(obs)).obs
    return ticks


def _device_loop(engine, policy, n: int):
    lf = policy if isinstance(policy, LaneFollower) else LaneFollower(obs_config=engine.obs_config)
    obs = engine.observe_device()
    alive = torch.as_tensor(engine.alive, device=engine.device)
    ticks = torch.zeros((), dtype=torch.int64, device=engine.device)
    for _ in range(n):
        ticks += alive.sum()
        out = engine.step(lf.on_device(engine, obs))
        obs, alive = out.obs, out.info["alive"]
    return int(ticks)


def measure_engine(engine, policy, steps: int, warmup: int, path: str = "vectorized") -> BenchReport:
    """``warmup`` untimed then ``steps`` timed closed-loop ticks of ``policy``
    on ``engine`` along ``path``; CASPS = alive agent-ticks / wall seconds."""
    if path not in PATHS:
        raise ValueError(f"unknown bench path {path!r} (have {PATHS})")
    loop = _host_loop if path == "vectorized" else _device_loop
    loop(engine, policy, warmup)
    engine.reset_phase_timers()
    torch.cuda.synchronize(engine.device)
    t0 = time.perf_counter()
    ticks = loop(engine, policy, steps)
    torch.cuda.synchronize(engine.device)
    wall = time.perf_counter() - t0
    return BenchReport(num_envs=engine.config.num_envs, num_agents=engine.config.num_agents,
                       backend=engine.config.dynamics_mode, path=path, casps=ticks / wall if wall > 0 else 0.0,
                       steps=steps, warmup_steps=warmup, wall_seconds=wall,
                       phase_ms={k: engine.phase_seconds[k] * 1000.0 / max(steps, 1) for k in PHASES},
                       workers=engine.config.effective_workers)


def _bench_engine(W: int, M: int, mode: str, seed: int, device):
    """The reference's collision-free bench fixture (one straight scene, three
    lanes, 8 m gaps): the alive population stays constant."""
    from .config import RootConfig, build_engine
    from .scenes import prepare_scene, straight_scene
    cfg = RootConfig()
    cfg.env.num_envs, cfg.env.num_agents_per_env, cfg.env.dynamics_mode, cfg.seed = W, M, mode, seed
    scene = prepare_scene(straight_scene("bench", agent_count=M, agent_gap=8.0, lane_offsets=(0.0, 4.0, -4.0),
                                         goal_dist=60.0))
    return build_engine(cfg, scenes=[scene], device=device)


def run_bench(grid: list, steps: int = 40, warmup: int = 8, mode: str = "dynamic", paths: tuple = PATHS,
              seed: int = 42, engine_factory=None, repeats: int = 1, device=None) -> list:
    """Every (W, M) of ``grid`` on every path; with ``repeats`` > 1 the runs
    interleave and the best CASPS per (W, M, path) is kept."""
    factory = engine_factory or (lambda W, M: _bench_engine(W, M, mode, seed, device))
    best: dict = {}
    for _ in range(repeats):
        for W, M in grid:
            for path in paths:
                eng = factory(W, M)
                # the reference scales smaller batches' step counts up to similar wall time
                n = steps * max(1, grid[-1][0] // max(W, 1))
                rep = measure_engine(eng, LaneFollower(obs_config=eng.obs_config), n, warmup, path=path)
                key = (W, M, path)
                if key not in best or rep.casps > best[key].casps:
                    best[key] = rep
    return [best[(W, M, p)] for W, M in grid for p in paths]


def write_bench_csv(reports: list, path) -> None:
    rows = [r.to_row() for r in reports]
    with open(path, "w", newline="", encoding="utf-8") as fh:
        out = csv.DictWriter(fh, fieldnames=list(rows[0]))
        out.writeheader()
        out.writerows(rows)
