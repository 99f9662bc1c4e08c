"""Kernel-time sweep: fused step at W x 16 over launch shapes (warps, CTAs/SM)."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

L2 = 126 << 20
shapes = [tuple(int(v) for v in x.split("x")) for x in sys.argv[2].split(",")]
for W in [int(x) for x in sys.argv[1].split(",")]:
    cfg = C.RootConfig()
    cfg.env.num_envs = W
    eng = Engine(**C.build_inputs(cfg).as_kwargs(), device=torch.device("cuda:0"))
    D = eng.obs_config.obs_dim
    ring = max(2, math.ceil(2 * L2 / (W * 16 * D * 4)))
    obs = torch.empty((ring, W, 16, D), device="cuda:0")
    bufs = [eng.new_step_buffers(obs[i]) for i in range(ring)]
    acts = torch.zeros((W, 16, 3), dtype=torch.float64, device="cuda:0")
    eng.observe(out=obs[ring - 1], as_numpy=False)
    for nw, cps in shapes:
        eng.tune(nw, cps)
        for i in range(10):
            eng.lane_follower(obs[(i - 1) % ring], out=acts)
            eng.launch_step(acts, bufs[i % ring], autoreset=True)
        n = 100
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        torch.cuda.synchronize()
        for i in range(n):
            eng.lane_follower(obs[(i - 1) % ring], out=acts)
            e0[i].record()
            eng.launch_step(acts, bufs[i % ring], autoreset=True)
            e1[i].record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in zip(e0, e1))
        med = ms[len(ms) // 2]
        gbs = W * 16 * 8184 / (med / 1e3) / 1e9
        print(f"W={W:5d} warps={nw:2d} ctas/SM={cps} kernel median {med*1e3:8.1f} us  min {ms[0]*1e3:8.1f}  "
              f"CASPS(kernel) {W*16/(med/1e3)/1e6:8.1f} M  {gbs:7.1f} GB/s", flush=True)
