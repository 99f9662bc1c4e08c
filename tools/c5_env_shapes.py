"""Launch shapes for the configs[4] env step (1024 x 16, one tick per launch, fused
LaneFollower, autoreset): device time per tick over a CUDA graph of 64 launches,
for (warps per world, CTAs per SM, mode) candidates.

  python tools/c5_env_shapes.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

dev = torch.device("cuda:0")
cfg = C.RootConfig()
cfg.env.num_envs = 1024
inp = C.build_inputs(cfg, device=dev)
shapes = [None, (4, 4, 0), (4, 6, 0), (4, 8, 0), (8, 2, 0), (7, 0, 2), (4, 3, 0), (2, 8, 0)]
for rep in range(2):
    for sh in shapes:
        eng = Engine(**inp.as_kwargs(), device=dev)
        try:
            if sh is not None:
                eng.tune(sh[0], sh[1], mode=sh[2])
        except Exception as e:  # noqa: BLE001
            print(sh, "rejected:", str(e)[:100])
            continue
        rb = eng.new_rollout_buffers(2)
        acts = torch.zeros((1024, 16, 3), dtype=torch.float64, device=dev)
        eng.observe(out=rb.obs[1], as_numpy=False, next_actions=acts)
        t = [0]

        def run(k):
            for _ in range(k):
                eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=1, ring_start=t[0] % 2)
                t[0] += 1
        run(4)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run(64)
        best = None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / 64
            best = us if best is None else min(best, us)
        print(f"{str(sh):14s} {eng.launch_shape()}: {best:7.2f} us/tick", flush=True)
        del eng, rb, g
        torch.cuda.empty_cache()
