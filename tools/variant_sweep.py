"""Kernel-variant sweep on the bench workload (LaneFollower fused, autoreset,
obs ring > L2): device time per tick for every (env knob setting, W, ticks per
launch) -- one process, engines rebuilt per setting.

  python tools/variant_sweep.py "DG_PIPE=1,DG_RESIDENT=1" "DG_PIPE=0,DG_RESIDENT=1" ...
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import _native as N  # noqa: E402

if os.environ.get("DG_LIB_PATH"):          # a variant build (tools/step_variants.py)
    N.LIB_PATH = Path(os.environ["DG_LIB_PATH"])
    N.load_library(build_if_missing=False)
from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

dev = torch.device("cuda:0")
settings = sys.argv[1:] or ["DG_PIPE=1,DG_RESIDENT=1"]
inputs = {}
for W in (256, 4096):
    cfg = C.RootConfig()
    cfg.env.num_envs = W
    inputs[W] = C.build_inputs(cfg, device=dev)
for st in settings:
    for kv in st.split(","):
        k, v = kv.split("=")
        os.environ[k] = v
    for W, R, n in ((256, 20, 10), (256, 64, 4), (4096, 64, 2)):
        eng = Engine(**inputs[W].as_kwargs(), device=dev)
        if W <= 296 and os.environ.get("SWEEP_SHAPE"):          # "warps:mode", e.g. 8:2
            nw, md = (int(v) for v in os.environ["SWEEP_SHAPE"].split(":"))
            eng.tune(nw, 0, mode=md)
        M, D = eng.M, eng.obs_config.obs_dim
        ring = max(2, -(-(300 << 20) // (W * M * D * 4)))
        rb = eng.new_rollout_buffers(ring)
        acts = torch.zeros((W, M, 3), dtype=torch.float64, device=dev)
        eng.observe(out=rb.obs[ring - 1], as_numpy=False, next_actions=acts)
        tick = [0]
        counters = torch.zeros((W, 5), dtype=torch.int32, device=dev) if os.environ.get("SWEEP_COUNT") else None

        def run(k):
            for _ in range(k):
                eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=R, ring_start=tick[0] % ring,
                                event_counts=counters)
                tick[0] += R
        run(2)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run(n)
        best = None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / (n * R)
            best = us if best is None else min(best, us)
        print(f"{st:32s} W={W:5d} R={R:3d} {eng.launch_shape()}: {best:7.2f} us/tick  "
              f"{W * M / best:7.1f} M agent-steps/s", flush=True)
        del eng, rb, g
        torch.cuda.empty_cache()
