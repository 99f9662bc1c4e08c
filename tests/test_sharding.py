"""Multi-GPU path on CPU: world sharding is exact (each shard reproduces the
same worlds of the global run bit for bit) and the one collective -- the
all-gather of per-rank episode counters -- works over a world-size-2 gloo
group (two processes, 127.0.0.1)."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from cases import cfg_of, philox_actions
from oracle import OracleEngine
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.params import EVENT_TYPES, STATE_FIELDS
from oracle.metrics import aggregate, drac_of_snapshot
from paper_2605_08528_b200.sharding import (allgather_metric_summaries, allgather_summaries, combine,
                                            combine_metrics, episode_summary, metric_summary,
                                            shard_inputs, shard_range)

W, M, T = 6, 16, 30


def _counts(out, counts):
    for i, k in enumerate(EVENT_TYPES):
        counts[:, i] += out.events[k].sum(axis=1)
    counts[:, 4] += out.info["alive_pre"].sum(axis=1)


def test_shard_range_partitions():
    for n in (1, 2, 3, 4, 8):
        ranges = [shard_range(4096, r, n) for r in range(n)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 4096
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_shards_reproduce_the_global_run():
    inp = C.build_inputs(cfg_of(W, M, seed=7))
    acts = philox_actions(2, T, W, M).astype(np.float64)
    full = OracleEngine(**inp.as_kwargs())
    shards = [OracleEngine(**shard_inputs(inp, r, 2).as_kwargs()) for r in range(2)]
    for t in range(T):
        o = full.step(acts[t])
        parts = [sh.step(acts[t][slice(*shard_range(W, r, 2))]) for r, sh in enumerate(shards)]
        assert np.array_equal(np.concatenate([p.obs for p in parts]), o.obs)
        assert np.array_equal(np.concatenate([p.rewards for p in parts]), o.rewards)
        for k in EVENT_TYPES:
            assert np.array_equal(np.concatenate([p.events[k] for p in parts]), o.events[k])
    for k in STATE_FIELDS:
        assert np.array_equal(np.concatenate([sh.state[k] for sh in shards]), full.state[k])


def _worker(rank, port, result_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    inp = C.build_inputs(cfg_of(W, M, seed=7))
    mine = shard_inputs(inp, rank, 2)
    eng = OracleEngine(**mine.as_kwargs())
    acts = philox_actions(2, T, W, M).astype(np.float64)
    lo, hi = shard_range(W, rank, 2)
    counts = np.zeros((hi - lo, 5), dtype=np.int64)
    acc = _MetricAcc(hi - lo)
    for t in range(T):
        out = eng.step(acts[t][lo:hi])
        _counts(out, counts)
        acc.add(out, eng)
    gathered = allgather_summaries(episode_summary(counts, int(eng.valid.sum())))
    mg = allgather_metric_summaries(acc.summary(eng.valid))
    if rank == 0:
        result_q.put((combine(gathered), combine_metrics(mg)))
    dist.destroy_process_group()


class _MetricAcc:
    def __init__(self, Wl):
        self.mx = np.zeros((Wl, M))
        self.goal = np.zeros((Wl, M), dtype=bool)
        self.coll = np.zeros((Wl, M), dtype=bool)

    def add(self, out, eng):
        self.mx = np.maximum(self.mx, drac_of_snapshot(out.info["state"], out.info["alive_pre"],
                                                       eng.r_hull, eng.d_hull))
        self.goal |= out.events["goal"]
        self.coll |= out.events["collision"]

    def summary(self, valid):
        return metric_summary(self.mx, valid, int((self.goal & valid).sum()), int((self.coll & valid).sum()),
                              threshold=0.0)


def test_gloo_allgather_of_episode_counters():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, got_m = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference of the same totals
    inp = C.build_inputs(cfg_of(W, M, seed=7))
    eng = OracleEngine(**inp.as_kwargs())
    acts = philox_actions(2, T, W, M).astype(np.float64)
    counts = np.zeros((W, 5), dtype=np.int64)
    acc = _MetricAcc(W)
    for t in range(T):
        out = eng.step(acts[t])
        _counts(out, counts)
        acc.add(out, eng)
    want = combine([episode_summary(counts, int(eng.valid.sum()))])
    assert got == want
    assert want["alive_ticks"] > 0
    # the gathered safety metrics equal the single-process episode_metrics reduction
    ref = aggregate(acc.goal, acc.coll, acc.mx, eng.valid, threshold=0.0)
    for k in ("goals", "collisions", "valid_agents", "sr", "cr"):
        assert got_m[k] == ref[k], k
    assert got_m["n_drac_over"] == int((acc.mx[eng.valid] > 0.0).sum()) > 0
    np.testing.assert_allclose(got_m["mean_max_drac"], ref["mean_max_drac"], rtol=1e-12)
