#!/usr/bin/env python
"""CASPS benchmark of the fused B200 vehicle step (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): 256 worlds x 16 agents, default
procedural pool (straight roads + crossroads, seed 42), dry road, dynamic
single-track backend.  A "step" = one fused env step (physics x4, 1929-dim
obs, rewards, events, tail) with the masked teleport reset of finished agents
fused in (autoreset, so the alive population stays at every valid slot) and
the LaneFollower bench policy fused in too (it reads the float32 ego block the
step just wrote and emits the next tick's actions) -- one kernel per tick.

  value   CASPS with everything resident in HBM; observations go to a rotating
          rollout ring larger than L2 (no cache reuse between steps)
  e2e     the same metric through the reference-facing numpy API
          (Engine.step with host arrays: H2D actions, D2H obs/rewards/dones/
          events/info every step, host LaneFollower: dg_lane_follower_rows)

N>1 (torchrun): 4096x16 worlds sharded by contiguous world range (BASELINE
configs[3]), no per-step communication; episode statistics all-gathered once
over NCCL after the timed region.  --impl reference times the CPU oracle
port (numpy restatement of the reference, all host threads).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
HEADLINE = (256, 16)
SCALE_TOTAL_WORLDS = 4096
REF_SAMPLE_WORLDS = 1024
DEFAULT_TICKS_PER_LAUNCH = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--worlds", type=int, default=0, help="override total worlds")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--cpu-steps", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the configs[3] single-GPU and configs[4] policy-rollout sub-lines")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly from the host (slower)")
    ap.add_argument("--shape", default="", help="launch shape '<warps>x<ctas/SM>' (default: the engine's choice)")
    ap.add_argument("--ticks-per-launch", type=int, default=0,
                    help="control ticks per persistent kernel launch (0 = default for the shape)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def root_config(total_worlds, M=16):
    from paper_2605_08528_b200 import config as C
    cfg = C.RootConfig()
    cfg.env.num_envs = total_worlds
    cfg.env.num_agents_per_env = M
    return cfg


def ring_slots(W, M, D):
    """Rollout-ring slots so the ring is > 2x L2 (obs never re-read from L2)."""
    return max(2, math.ceil(2 * L2_BYTES / (W * M * D * 4)))


def bench_config(W, M, D=1929):
    """The workload description, identical in both arms' lines."""
    ring = ring_slots(W, M, D)
    return {"workload": f"{W}x{M} default procedural pool (seed 42), dry, dynamic, LaneFollower policy, "
                        "finished agents teleported back to their start (autoreset)",
            "worlds": W, "agents": M, "obs_dim": D, "seed": 42, "policy": "LaneFollower", "autoreset": True,
            "l2": f"GPU arm: obs rotate through a {ring}-slot rollout ring "
                  f"({ring * W * M * D * 4 / 2**20:.0f} MiB > L2)"}


def shard_inputs(cfg, rank, world_size, dev=None):
    """This rank's contiguous world range of the global batch.  With ``dev`` the
    worlds are built on that GPU (worldgen.py: each rank builds only its shard,
    bit-identical to the same worlds of the whole batch); without, on the host."""
    from paper_2605_08528_b200 import config as C
    from paper_2605_08528_b200.sharding import shard_inputs as _shard
    return _shard(C.build_inputs(cfg, device=dev), rank, world_size)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(W, M, ticks):
    """dram read+write bytes of one launch of exactly this shape and tick
    count from a committed ncu --set full capture (profiles/ncu_traffic.json,
    key "WxMxticks"), or None -- never extrapolated from another tick count."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    rec = json.loads(p.read_text()).get(f"{W}x{M}x{ticks}")
    return None if rec is None else (float(rec["traffic_bytes"]), rec.get("source", ""))


def algorithmic_bytes_per_agent(obs_dim: int) -> int:
    """Bytes one agent-step must move to/from HBM, SURVEY.md §8(d):
    B = 4*obs_dim (obs row) + 12 (actions) + 96 (12 fp32 state in + out) + 4
    (reward) + 1 (done) + 4 (events) + 1 (reason) + 1 (alive) = 7,835 B at the
    1,929-float observation.  (The engine keeps its state in float64, so it moves
    more than the state term here; the obs row dominates either way.)"""
    return 4 * obs_dim + 12 + 96 + 4 + 1 + 4 + 1 + 1


def unmodified_reference(W, M, steps, warmup, cores):
    """The reference package itself (installed unmodified in baseline/_ref by
    pip), through its own harness: metrics.measure_engine
    (metrics.py:158-184) on build_engine(cfg) with the LaneFollower -- the
    vectorized path on every host thread (engine.py:258-270) over the same
    W x M batch, and the scalar reference_step path (engine.py:423-595) on a
    16-world sample.  measure_engine counts alive agents before each step
    and does not reset finished agents."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "drivegrid").is_dir():
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref /root/reference)"}
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    from drivegrid.config import RootConfig as RefRoot
    from drivegrid.config import build_engine as ref_build
    from drivegrid.metrics import measure_engine
    from drivegrid.policies import LaneFollower as RefLF

    out = {}
    for path, Wp, n, wu in (("vectorized", W, steps, warmup), ("scalar", min(W, 16), max(2, steps // 8), 1)):
        cfg = RefRoot()
        cfg.env.num_envs, cfg.env.num_agents_per_env = Wp, M
        cfg.env.num_workers = cores if path == "vectorized" else 0
        eng = ref_build(cfg)
        rep = measure_engine(eng, RefLF(obs_config=eng.obs_config), n, wu, reference=path == "scalar")
        out[path] = {"value": rep.casps, "unit": "agent-steps/s", "cores": rep.workers, "kind": "reference",
                     "sample": f"{Wp}x{M} default pool, {n} steps after {wu} warmup ({rep.wall_seconds:.1f} s), "
                               f"drivegrid.metrics.measure_engine(path={path!r}), unmodified reference "
                               f"(baseline/_ref), numpy {np.__version__}",
                     "phase_ms": {k: round(v, 3) for k, v in rep.phase_ms.items()}}
    return out


def run_reference(args, rank, world_size):
    """CPU oracle port (reference algorithm) on this host's cores."""
    if rank != 0:
        return
    from oracle import OracleEngine
    from paper_2605_08528_b200 import config as C
    from paper_2605_08528_b200.policies import LaneFollower

    cores = len(os.sched_getaffinity(0))
    W = args.worlds or (HEADLINE[0] if world_size == 1 else SCALE_TOTAL_WORLDS)
    cfg = root_config(W)
    inp = C.build_inputs(cfg)
    # bounded sample: the first REF_SAMPLE_WORLDS worlds of the (globally built)
    # batch per step, so a K-step run stays within minutes at 4096 worlds; CASPS
    # is per agent-tick, and the numpy path's per-agent cost is flat at this size
    Ws = min(W, REF_SAMPLE_WORLDS)
    if Ws < W:
        from paper_2605_08528_b200.sharding import shard_inputs as _shard
        inp = _shard(inp, 0, W // Ws)
    eng = OracleEngine(**inp.as_kwargs(), num_workers=cores)
    pol = LaneFollower(obs_config=eng.obs_config)
    obs = eng.observe()
    for _ in range(args.warmup):
        out = eng.step(pol(obs))
        eng.teleport_reset(out.dones)
        obs = out.obs
    ticks = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ticks += int(eng.alive.sum())
        out = eng.step(pol(obs))
        eng.teleport_reset(out.dones)
        obs = out.obs
    wall = time.perf_counter() - t0
    v = ticks / wall
    line = {
        "impl": "reference", "metric": "CASPS", "value": v, "unit": "agent-steps/s",
        "n_gpus": world_size, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "weak" if world_size == 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(W, 16),
        "cpu_baseline": {"value": v, "unit": "agent-steps/s", "cores": cores, "kind": "port",
                         "sample": f"{Ws} of the {W} worlds x16 (contiguous range 0..{Ws - 1}), {args.steps} steps "
                                   f"after {args.warmup} warmup, oracle/ numpy port, numpy {np.__version__}"},
        "e2e": {"value": v, "unit": "agent-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu:
        line["reference_package"] = unmodified_reference(W if world_size == 1 else HEADLINE[0], 16,
                                                         min(args.steps, 20), min(args.warmup, 3), cores)
    print(json.dumps(line), flush=True)


def cpu_baseline(steps):
    from oracle import OracleEngine
    from paper_2605_08528_b200 import config as C
    from paper_2605_08528_b200.policies import LaneFollower

    cores = len(os.sched_getaffinity(0))
    inp = C.build_inputs(root_config(HEADLINE[0]))
    eng = OracleEngine(**inp.as_kwargs(), num_workers=cores)
    pol = LaneFollower(obs_config=eng.obs_config)
    obs = eng.observe()
    for _ in range(2):
        out = eng.step(pol(obs))
        eng.teleport_reset(out.dones)
        obs = out.obs
    ticks, t0 = 0, time.perf_counter()
    for _ in range(steps):
        ticks += int(eng.alive.sum())
        out = eng.step(pol(obs))
        eng.teleport_reset(out.dones)
        obs = out.obs
    wall = time.perf_counter() - t0
    return {"value": ticks / wall, "unit": "agent-steps/s", "cores": cores, "kind": "port",
            "sample": f"256x16 default pool, LaneFollower+autoreset, {steps} steps after 2 warmup "
                      f"({wall:.1f} s), oracle/ numpy port, numpy {np.__version__}"}


def main():
    args = parse()
    rank, local_rank, world_size = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world_size)
        return
    import torch
    import torch.distributed as dist

    # DG_BENCH_DIST_BACKEND=gloo + DG_BENCH_ONE_DEVICE=1 exercise the N-rank code
    # path with every rank on cuda:0 (a one-GPU box); the real runs use NCCL
    backend = os.environ.get("DG_BENCH_DIST_BACKEND", "nccl")
    gpu = 0 if os.environ.get("DG_BENCH_ONE_DEVICE") == "1" else local_rank
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world_size > 1:
        if backend == "nccl":
            # NCCL logs its communicator (rank count, transports) to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else torch.device("cpu")   # collective tensors

    from paper_2605_08528_b200.engine import Engine

    W_total = args.worlds or (HEADLINE[0] if world_size == 1 else SCALE_TOTAL_WORLDS)
    inp = shard_inputs(root_config(W_total), rank, world_size, dev)
    eng = Engine(**inp.as_kwargs(), device=dev)
    if args.shape:
        nw, cps = (int(v) for v in args.shape.split("x"))
        eng.tune(nw, cps)
    W, M, D = eng.W, eng.M, eng.obs_config.obs_dim
    obs_bytes = W * M * D * 4
    ring = ring_slots(W_total, M, D) if world_size == 1 else ring_slots(W, M, D)
    # every tick writes its own ring slot (obs + the per-tick aux outputs)
    rbufs = eng.new_rollout_buffers(ring)
    R = args.ticks_per_launch or DEFAULT_TICKS_PER_LAUNCH
    # the LaneFollower is fused into the step: a launch reads actions (tick 0),
    # feeds the policy's actions to its later ticks through shared memory and
    # leaves the next launch's actions in next_actions (in place: a world's
    # CTA reads its rows before it overwrites them)
    acts = torch.zeros((W, M, 3), dtype=torch.float64, device=dev)
    eng.observe(out=rbufs.obs[ring - 1], as_numpy=False, next_actions=acts)
    stream = torch.cuda.current_stream(dev)

    # per-world episode counters on the device: goal/collision/crash/lane_forbidden
    # events and alive agent-ticks (the CASPS numerator, counted before each tick)
    counters = torch.zeros((W, 5), dtype=torch.int32, device=dev)
    tick = [0]
    tick_log = []          # ticks of every launch issued, in order

    def run_ticks(n, count=True):
        """n control ticks in ceil(n / R) launches of up to R ticks each."""
        done = 0
        while done < n:
            r = min(R, n - done)
            eng.launch_step(acts, rbufs, autoreset=True, next_actions=acts, ticks=r,
                            ring_start=tick[0] % ring, event_counts=counters if count else None)
            tick_log.append(r)
            tick[0] += r
            done += r

    # warm-up (untimed)
    run_ticks(args.warmup, count=False)
    torch.cuda.synchronize()
    valid_count = int(eng.valid.sum())
    assert int(eng.alive.sum()) == valid_count

    # The K timed ticks are captured once into a CUDA graph (outside the timed
    # region) so the device runs the launches back to back with no host gaps.
    # The per-launch kernel time (the roofline numerator) comes from a second
    # graph of the same launches without the counters, timed right after.
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eng.launches
    graph = None
    graph_ticks = []
    # device-side bracket of the K ticks: event-record nodes captured inside the
    # graph (cudaEventRecordExternal) fire when the device reaches them, so the
    # host's graph-submission latency before the first launch is not booked as
    # step time; the host-bracketed time is reported beside it (ms_incl_submit)
    g_start = torch.cuda.Event(enable_timing=True, external=True)
    g_stop = torch.cuda.Event(enable_timing=True, external=True)
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        n0 = len(tick_log)
        with torch.cuda.graph(graph):
            g_start.record()
            run_ticks(args.steps)
            g_stop.record()
        graph_ticks = tick_log[n0:]
        launches0 = eng.launches - len(graph_ticks)   # the captured launches run at replay
    if world_size > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        start.record(stream)
        if graph is not None:
            graph.replay()
        else:
            run_ticks(args.steps)
        stop.record(stream)
        torch.cuda.synchronize()
    launches = eng.launches - launches0
    launch_ticks = list(tick_log[len(tick_log) - launches:]) if graph is None else list(graph_ticks)
    total_ms = start.elapsed_time(stop)
    ms_incl_submit = total_ms
    if graph is not None:
        total_ms = g_start.elapsed_time(g_stop)
    if world_size > 1:
        t = torch.tensor([total_ms], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    n_launch = len(launch_ticks)
    assert sum(launch_ticks) == args.steps, (launch_ticks, args.steps)
    if graph is not None:
        g_step = torch.cuda.CUDAGraph()
        k0 = torch.cuda.Event(enable_timing=True, external=True)
        k1 = torch.cuda.Event(enable_timing=True, external=True)
        with torch.cuda.graph(g_step):
            k0.record()
            run_ticks(args.steps, count=False)
            k1.record()
        torch.cuda.synchronize()
        g_step.replay()
        torch.cuda.synchronize()
        kern_total = k0.elapsed_time(k1)
    else:
        kern_total = total_ms
    kern_avg = kern_total / n_launch            # ms per launch
    ticks_per_launch = args.steps / n_launch
    from paper_2605_08528_b200.sharding import allgather_summaries, combine, episode_summary
    local = episode_summary(counters.cpu().numpy(), valid_count)
    # episode statistics: the only cross-rank traffic (one NCCL all-gather)
    totals = combine(allgather_summaries(local) if world_size > 1 else [local])
    agent_ticks = totals["alive_ticks"]          # alive agents before each timed tick, device-counted
    value = agent_ticks / (total_ms / 1e3)

    # e2e through the numpy API on every rank at once; whole-job value =
    # all ranks' agent-ticks / the slowest rank's wall time
    e2e_steps = args.e2e_steps or 200
    if world_size > 1:
        dist.barrier()
    e2e = e2e_numpy(eng, e2e_steps)
    if world_size > 1:
        t = torch.tensor([float(e2e["ticks"]), e2e["wall_s"], float(e2e["h2d_bytes_per_step"]),
                          float(e2e["d2h_bytes_per_step"])], dtype=torch.float64, device=cdev)
        parts = [torch.empty_like(t) for _ in range(world_size)]
        dist.all_gather(parts, t)
        parts = torch.stack(parts).cpu().numpy()
        e2e["ticks"] = int(parts[:, 0].sum())
        e2e["wall_s"] = float(parts[:, 1].max())
        e2e["value"] = e2e["ticks"] / e2e["wall_s"]
        e2e["h2d_bytes_per_step"] = int(parts[:, 2].sum())
        e2e["d2h_bytes_per_step"] = int(parts[:, 3].sum())
        e2e["ranks"] = world_size

    if rank == 0:
        peak, peak_src = measured_peaks()
        per_agent = algorithmic_bytes_per_agent(D)
        achieved = per_agent * W * M * ticks_per_launch / (kern_avg / 1e3) / 1e9
        uniform = len(set(launch_ticks)) == 1
        traffic = ncu_traffic(W, M, launch_ticks[0]) if (world_size == 1 and uniform) else None
        line = {
            "metric": "CASPS", "value": value, "unit": "agent-steps/s", "n_gpus": world_size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if world_size == 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(W_total, M, D),
            "launch": {"launches": n_launch, "ticks_per_launch": launch_ticks[0] if uniform else launch_ticks,
                       "max_ticks_per_launch": R, "cuda_graph": graph is not None,
                       "timing": ("CUDA events captured inside the graph (cudaEventRecordExternal): device time "
                                  "from the first launch of the K ticks to the end of the last; barrier + "
                                  "synchronize around the replay" if graph is not None else
                                  "CUDA events around the launches on the launching stream"),
                       "ms_incl_submit": ms_incl_submit,
                       "ring_slots": ring, "kernel_shape": eng.launch_shape(),
                       "obs_clear": "resident ring (DgStepIO.obs_resident): a slot keeps its zero background, "
                                    "a tick clears only the row spans its new content no longer covers",
                       "parallelism": f"world-shard x{world_size}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None if traffic is None else traffic[0],
                         "traffic_source": None if traffic is None else traffic[1],
                         "algorithmic_bytes_per_launch": per_agent * W * M * ticks_per_launch,
                         "bytes_per_agent_step": per_agent, "kernel_ms": kern_avg,
                         "kernel_ms_per_tick": kern_avg / ticks_per_launch,
                         "peak_source": peak_src},
            "gpu_launches": launches,
            "episode_counters": totals,
        }
        line["clocks"] = clk.summary()
        line["e2e"] = e2e
        if not args.no_c5 and world_size == 1:
            line["c5_policy_rollout"] = bench_c5(dev)
        if not args.no_c5 and world_size == 1:
            line["c4_single_gpu"] = bench_c4(dev, steps=max(64, args.steps), R=R)
        if not args.no_cpu and world_size == 1:
            line["cpu_baseline"] = cpu_baseline(args.cpu_steps or 40)
            line["reference_package"] = unmodified_reference(W_total, M, 20, 3, len(os.sched_getaffinity(0)))
        print(json.dumps(line), flush=True)
    if world_size > 1:
        dist.destroy_process_group()


def bench_c4(dev, steps=200, R=DEFAULT_TICKS_PER_LAUNCH, W=SCALE_TOTAL_WORLDS, M=16):
    """BASELINE configs[3] at N=1: the 4096 x 16 batch the multi-GPU runs shard
    (the N-GPU lines divide these worlds), timed exactly like the headline:
    fused LaneFollower + autoreset, persistent launches of R ticks, one CUDA
    graph, obs ring > L2, device-counted alive agent-ticks."""
    import torch
    from paper_2605_08528_b200.engine import Engine

    eng = Engine(**shard_inputs(root_config(W, M), 0, 1, dev).as_kwargs(), device=dev)
    D = eng.obs_config.obs_dim
    ring = max(2, math.ceil(2 * L2_BYTES / (W * M * D * 4)))
    rb = eng.new_rollout_buffers(ring)
    acts = torch.zeros((W, M, 3), dtype=torch.float64, device=dev)
    eng.observe(out=rb.obs[ring - 1], as_numpy=False, next_actions=acts)
    counters = torch.zeros((W, 5), dtype=torch.int32, device=dev)
    tick = [0]

    def run(n, count):
        done = 0
        while done < n:
            r = min(R, n - done)
            eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=r, ring_start=tick[0] % ring,
                            event_counts=counters if count else None)
            tick[0] += r
            done += r

    run(2 * R, False)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run(steps, True)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ticks = int(counters[:, 4].sum().item())
    return {"metric": "CASPS", "value": ticks / (ms / 1e3), "unit": "agent-steps/s", "n_gpus": 1,
            "workload": f"{W}x{M} default pool (the batch the N-GPU runs shard), LaneFollower + autoreset",
            "steps": steps, "ms_per_step": ms / steps, "ticks_per_launch": R}


def policy_flops_per_agent(n_road: float, n_veh: float, ego_dim: int = 11, nets: int = 2) -> float:
    """Algorithmic FLOPs of one policy forward per agent (App. E network,
    policy.py): only VALID road / vehicle slots count (masked max-pool
    ignores the rest); 2 FLOP per MAC; actor + critic."""
    per_net = (n_road * (5 * 96 + 96 * 96) + n_veh * (7 * 96 + 96 * 96)
               + ego_dim * 64 + 64 * 64 + 256 * 128 + 128 * 64)
    return 2.0 * nets * per_net + 2.0 * 64 * (3 + 1)


def bench_c5(dev, ticks=128, W=1024, M=16, reps=2):
    """BASELINE configs[4]: 1024 x 16 rollout of T=128 ticks with the policy
    MLP (actor mean -> next actions, critic values) fused into the loop on
    the device: per tick one step launch + two tcgen05 policy launches, the
    whole rollout one CUDA graph.  Returns a dict for the JSON line."""
    import torch
    from paper_2605_08528_b200.engine import Engine
    from paper_2605_08528_b200.policy import PolicyMLP

    inp = shard_inputs(root_config(W, M), 0, 1, dev)
    eng = Engine(**inp.as_kwargs(), device=dev)
    D = eng.obs_config.obs_dim
    pol = PolicyMLP(eng.obs_config, seed=0, device=dev, head_scale=1.0)
    rb = eng.new_rollout_buffers(ticks)          # [T][W][M][D]: 1 GB > L2, every tick its own slot
    values = torch.empty((ticks, W, M), dtype=torch.float32, device=dev)
    log_probs = torch.empty((ticks, W, M), dtype=torch.float32, device=dev)
    actions_out = torch.empty((ticks, W, M, 3), dtype=torch.float32, device=dev)
    ppo = dict(sample=True, seed=1234, log_probs=log_probs, actions_out=actions_out)
    from paper_2605_08528_b200.policy import gae
    acts = torch.zeros((W, M, 3), dtype=torch.float64, device=dev)
    acts[..., 0] = 0.5
    counters = torch.zeros((W, 5), dtype=torch.int32, device=dev)
    # warm-up (allocates the policy scratch, packs the weights)
    eng.run_mlp_ticks(acts, rb, pol, 4, autoreset=True, values=values, **ppo)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    launches0 = eng.launches
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        # the PPO collection: T ticks of (step -> sampled actions, log-probs, values),
        # then GAE over the T-1 complete transitions
        eng.run_mlp_ticks(acts, rb, pol, ticks, autoreset=True, values=values, event_counts=counters, **ppo)
        adv, ret = gae(rb.views["rewards"][1:], rb.views["dones"][1:], values, 0.99, 0.98)
    launches = eng.launches - launches0 + 1
    g.replay()
    torch.cuda.synchronize()
    counters.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    alive_ticks = int(counters[:, 4].sum().item()) / reps
    # the two halves of a tick, each timed alone over the same T ticks
    obs_last = rb.obs[ticks - 1]
    gp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gp):
        for _ in range(ticks):
            pol.forward(obs_last, actions=acts, value=values[0], sample=True, seed=1, log_prob=log_probs[0],
                        actions_f32=actions_out[0])
    ge = torch.cuda.CUDAGraph()
    with torch.cuda.graph(ge):
        for t in range(ticks):
            eng.launch_step(acts, rb, autoreset=True, ticks=1, ring_start=t)
    res = {}
    for name, gg in (("policy", gp), ("env", ge)):
        gg.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        gg.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / ticks
    oc = eng.obs_config
    road = obs_last[..., oc.ego_dim:oc.ego_dim + 5 * oc.k_road].reshape(W, M, oc.k_road, 5)
    veh = obs_last[..., oc.ego_dim + 5 * oc.k_road:].reshape(W, M, oc.k_vehicles, 7)
    n_road = float(((road[..., 3] != 0) | (road[..., 4] != 0)).sum(-1).float().mean())
    n_veh = float((veh[..., 2] != 0).sum(-1).float().mean())
    flops = policy_flops_per_agent(n_road, n_veh, oc.ego_dim) * W * M
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops_sustained"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 1400.0
    achieved = flops / (res["policy"] / 1e3) / 1e12
    return {"metric": "CASPS", "value": alive_ticks / (ms / 1e3), "unit": "agent-steps/s",
            "workload": f"{W}x{M} default pool, T={ticks} PPO rollout: policy MLP fused into the loop "
                        "(actor sample + log-prob, critic value: step + 2 tcgen05 launches per tick), "
                        "autoreset, GAE at the end, one CUDA graph",
            "ms_per_tick": ms / ticks, "env_ms_per_tick": res["env"], "policy_ms_per_tick": res["policy"],
            "gpu_launches": launches, "launches_per_tick": launches / ticks,
            "valid_slots_per_agent": {"road": n_road, "vehicle": n_veh},
            "policy_roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                                "frac": achieved / peak, "flops_per_agent": flops / (W * M),
                                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"}}


def e2e_numpy(eng, steps):
    """The reference-facing call: numpy actions in, numpy StepOutput out."""
    import torch
    from paper_2605_08528_b200.policies import LaneFollower

    pol = LaneFollower(obs_config=eng.obs_config)
    obs = eng.observe()
    for _ in range(3):
        out = eng.step(pol(obs), autoreset=True)
        obs = out.obs
    torch.cuda.synchronize()
    obs_bytes0 = int(eng.d2h_bytes.item())
    launches0 = eng.launches
    ticks = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        out = eng.step(pol(obs), autoreset=True)
        ticks += int(out.info["alive_pre"].sum())     # alive before the step (measure_engine)
        obs = out.obs
    wall = time.perf_counter() - t0
    W, M, D = eng.W, eng.M, eng.obs_config.obs_dim
    obs_bytes = (int(eng.d2h_bytes.item()) - obs_bytes0) / steps
    aux_bytes = int(eng._host_blob.numel()) - eng._host_obs_bytes
    return {"value": ticks / wall, "unit": "agent-steps/s", "h2d_bytes_per_step": W * M * 3 * 8,
            "d2h_bytes_per_step": int(round(obs_bytes)) + aux_bytes,
            "d2h_detail": {"obs_prefix_bytes_per_step": obs_bytes, "obs_dense_bytes": W * M * D * 4,
                           "aux_bytes_per_step": aux_bytes,
                           "note": "the obs rows reach the numpy array bit-exact; only each row's non-zero "
                                   "road / vehicle prefix (and zeros over a shorter prefix than the slab "
                                   "held) crosses PCIe, written by the device into mapped pinned slabs"},
            "gpu_launches": eng.launches - launches0,
            "steps": steps, "ticks": ticks, "wall_s": wall,
            "ms_per_step": 1e3 * wall / steps, "host_slabs": eng._mapped_pool.slabs,
            "api": "Engine.step(numpy actions) -> numpy StepOutput, autoreset, host LaneFollower (dg_lane_follower_rows, the numpy expression bit for bit); "
                   "alive agents counted before each step (metrics.py:168-170)"}


if __name__ == "__main__":
    main()
