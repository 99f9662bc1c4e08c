"""bench.py's N-rank path (BASELINE configs[3]: 4096 x 16 sharded by world,
no per-step communication, episode statistics gathered once after the timed
region) run under torchrun with 2 and 4 ranks on this one GPU (gloo for the
collectives, every rank on cuda:0): the gathered counters -- events and the
alive agent-ticks CASPS is computed from -- equal the single-rank run's.
SURVEY.md section 8(e); the reference fans worlds out over threads
(engine.py:262-270)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
ARGS = ["--steps", "16", "--warmup", "3", "--no-cpu", "--no-c5", "--e2e-steps", "3", "--worlds", "4096"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(n: int) -> dict:
    env = dict(os.environ, DG_BENCH_DIST_BACKEND="gloo", DG_BENCH_ONE_DEVICE="1")
    if n == 1:
        cmd = [sys.executable, "bench.py", "--gpus", "1", *ARGS]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(n),
               *ARGS]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]          # rank 0 alone prints
    return json.loads(lines[0])


def test_sharded_bench_counters_equal_single_rank():
    one = _run(1)
    assert one["episode_counters"]["alive_ticks"] == 4096 * 16 * 16
    for n in (2, 4):
        line = _run(n)
        assert line["n_gpus"] == n
        assert line["launch"]["parallelism"] == f"world-shard x{n}"
        assert line["episode_counters"] == one["episode_counters"], n
        assert line["e2e"]["ranks"] == n
