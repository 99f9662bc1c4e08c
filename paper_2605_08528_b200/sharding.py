"""World sharding across GPUs (one process per GPU).

Worlds are independent -- no query crosses a world (engine.py:177-183,
observation.py:239-240) -- so rank r of N owns the contiguous world range
[r*W/N, (r+1)*W/N).  The host tables are built for ALL worlds first (scene
assignment on Philox stream (seed, 0), weather on (seed, 2)) and then sliced,
which keeps every shard bit-identical to the same worlds of a one-GPU run.

There is no per-step communication.  Episode counters (goal, collision,
crash, lane_forbidden, alive agent-ticks per world; see DgStepIO.event_counts)
are reduced per rank and all-gathered once per episode / bench window; the
rank-ordered host sum keeps SR/CR exact and deterministic.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

from .params import SimConfig
from .scenes import WorldBatch


def shard_range(W: int, rank: int, world_size: int) -> tuple[int, int]:
    return rank * W // world_size, (rank + 1) * W // world_size


def shard_worlds(worlds: WorldBatch, lo: int, hi: int) -> WorldBatch:
    if hasattr(worlds, "shard"):
        return worlds.shard(lo, hi)       # DeviceWorldBatch: the rank builds only its worlds
    sl = slice(lo, hi)
    return WorldBatch(worlds.midpoints[sl], worlds.directions[sl], worlds.type_codes[sl],
                      worlds.half_lengths[sl], worlds.half_widths[sl], worlds.mask[sl],
                      worlds.grid_offsets[sl], worlds.scenario_ids[sl],
                      scene_index=None if worlds.scene_index is None else worlds.scene_index[sl],
                      scene_tables=worlds.scene_tables)


def shard_inputs(inputs, rank: int, world_size: int):
    """EngineInputs of this rank's world range (a shallow copy)."""
    if world_size == 1:
        return inputs
    W = inputs.sim.num_envs
    lo, hi = shard_range(W, rank, world_size)
    out = replace(inputs)
    out.worlds = shard_worlds(inputs.worlds, lo, hi)
    out.assignment = np.asarray(inputs.assignment)[lo:hi]
    out.frictions = list(inputs.frictions[lo:hi])
    out.sim = replace(inputs.sim, num_envs=hi - lo) if isinstance(inputs.sim, SimConfig) else inputs.sim
    return out


COUNTER_NAMES = ("goal", "collision", "crash", "lane_forbidden", "alive_ticks")


def episode_summary(counts: np.ndarray, valid_agents: int) -> dict:
    """Totals of the per-world counters [W][5] (any rank's or the gathered sum)."""
    tot = np.asarray(counts, dtype=np.int64).reshape(-1, 5).sum(axis=0)
    out = {k: int(v) for k, v in zip(COUNTER_NAMES, tot)}
    out["valid_agents"] = int(valid_agents)
    return out


def allgather_summaries(local: dict, group=None) -> list:
    """Rank-ordered list of every rank's summary (one all_gather of int64s;
    NCCL on GPU ranks, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    keys = (*COUNTER_NAMES, "valid_agents")
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([local[k] for k in keys], dtype=torch.int64, device=dev)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return [{k: int(v) for k, v in zip(keys, p.cpu().tolist())} for p in parts]


def combine(summaries: list) -> dict:
    keys = (*COUNTER_NAMES, "valid_agents")
    tot = {k: sum(s[k] for s in summaries) for k in keys}
    tot["success_rate_events"] = tot["goal"] / tot["valid_agents"] if tot["valid_agents"] else 0.0
    tot["collision_rate_events"] = tot["collision"] / tot["valid_agents"] if tot["valid_agents"] else 0.0
    return tot


# ---------------------------------------------------------------- safety metrics
METRIC_INT_KEYS = ("valid_agents", "goals", "collisions", "n_drac_over")


def metric_summary(per_agent_max_drac, valid, goals: int, collisions: int, threshold: float = 3.4) -> dict:
    """Sufficient statistics of one rank's episode metrics (metrics.py:110-125):
    goal / collision agent counts, valid agents, and the count and sum of the
    per-agent peak DRACs over ``threshold``."""
    valid = np.asarray(valid, dtype=bool)
    over = np.asarray(per_agent_max_drac)[valid & (np.asarray(per_agent_max_drac) > threshold)]
    return {"valid_agents": int(valid.sum()), "goals": int(goals), "collisions": int(collisions),
            "n_drac_over": int(over.size), "sum_drac_over": float(over.sum())}


def allgather_metric_summaries(local: dict, group=None) -> list:
    """Rank-ordered metric summaries: one all_gather of four int64 counts and
    one of the float64 DRAC sum (NCCL on GPU ranks, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    n = dist.get_world_size(group)
    ti = torch.tensor([local[k] for k in METRIC_INT_KEYS], dtype=torch.int64, device=dev)
    tf = torch.tensor([local["sum_drac_over"]], dtype=torch.float64, device=dev)
    pi = [torch.empty_like(ti) for _ in range(n)]
    pf = [torch.empty_like(tf) for _ in range(n)]
    dist.all_gather(pi, ti, group=group)
    dist.all_gather(pf, tf, group=group)
    out = []
    for a, b in zip(pi, pf):
        d = {k: int(v) for k, v in zip(METRIC_INT_KEYS, a.cpu().tolist())}
        d["sum_drac_over"] = float(b.cpu().item())
        out.append(d)
    return out


def combine_metrics(summaries: list) -> dict:
    """SR / CR / mean peak DRAC of the whole job from rank-ordered summaries
    (the rank order fixes the float summation order: deterministic)."""
    tot = {k: sum(s[k] for s in summaries) for k in METRIC_INT_KEYS}
    sdr = 0.0
    for s in summaries:
        sdr += s["sum_drac_over"]
    n = tot["valid_agents"]
    return {"sr": tot["goals"] / n if n else 0.0, "cr": tot["collisions"] / n if n else 0.0,
            "mean_max_drac": sdr / tot["n_drac_over"] if tot["n_drac_over"] else 0.0, **tot}
