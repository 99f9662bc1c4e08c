"""Kernel-time sweep of the fused step at W x 16 over launch shapes, timed on
the device with CUDA graphs (no host launch overhead inside the timed region).

shape syntax: "<warps>x<ctas/SM>" (fused) or "s<agents/CTA>x<ctas/SM>" (split)."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

L2 = 126 << 20


def parse_shape(x):
    mode = 1 if x.startswith("s") else 0
    nw, cps = (int(v) for v in x.lstrip("s").split("x"))
    return nw, cps, mode


shapes = [parse_shape(x) for x in sys.argv[2].split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
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
    for nw, cps, mode in shapes:
        eng.tune(nw, cps, mode=mode)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for i in range(3):  # warm-up outside the graph
                eng.lane_follower(obs[(i - 1) % ring], out=acts)
                eng.launch_step(acts, bufs[i % ring], autoreset=True)
        torch.cuda.synchronize()
        g_full, g_step = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_full):
            for i in range(steps):
                eng.lane_follower(obs[(i - 1) % ring], out=acts)
                eng.launch_step(acts, bufs[i % ring], autoreset=True)
        with torch.cuda.graph(g_step):
            for i in range(steps):
                eng.launch_step(acts, bufs[i % ring], autoreset=True)
        res = {}
        for name, g in (("policy+step", g_full), ("step only", g_step)):
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(5):
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / steps)
            res[name] = best
        st = res["step only"]
        gbs = W * 16 * 8184 / (st / 1e3) / 1e9
        print(f"W={W:5d} {'split' if mode else 'fused'} warps={nw:2d} ctas/SM={cps}  step {st*1e3:7.1f} us "
              f"(+policy {res['policy+step']*1e3:7.1f} us)  CASPS {W*16/(res['policy+step']/1e3)/1e6:7.1f} M  "
              f"{gbs:7.1f} GB/s", flush=True)
