"""Per-tick device time on the dense 73-lane scene (6,000 segments: too large
for shared memory, so the geometry is read in place from global memory -- by
the fused kernel's global-geometry variant, or the split kernels) next to the
default pool at the same batch, all device-resident LaneFollower loops in one
CUDA graph of 32 ticks."""
import sys
from pathlib import Path

sys.path[:0] = [str(Path(__file__).resolve().parents[1]), str(Path(__file__).resolve().parents[1] / "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import cfg_of  # noqa: E402
from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402
from paper_2605_08528_b200.scenes import prepare_scene, straight_scene  # noqa: E402

dev = torch.device("cuda:0")
W, M, T = 256, 8, 32
lanes = tuple(float(x) for x in np.round(np.arange(-9.0, 9.01, 0.25), 2))
dense = prepare_scene(straight_scene("dense", lane_offsets=lanes, agent_count=M, agent_gap=15.0, goal_dist=40.0))
for name, scenes, kw in (("default pool, fused", None, {}), ("default pool, split", None, {"launch_mode": 1}),
                         ("dense 73-lane, global, fused", [dense], {}),
                         ("dense 73-lane, global, fused 4x4", [dense], {"launch_mode": 0, "warps_per_world": 4}),
                         ("dense 73-lane, global, split", [dense], {"launch_mode": 1})):
    eng = Engine(**C.build_inputs(cfg_of(W, M, seed=3), scenes=scenes).as_kwargs(), device=dev, **kw)
    a = eng.lane_follower(eng.observe_device())
    split = eng.launch_shape()["mode"] == "split"
    res = []
    for R in ((1,) if split else (1, T)):
        bufs = eng.new_step_buffers() if R == 1 else eng.new_rollout_buffers(2)
        for _ in range(3):
            eng.launch_step(a, bufs, autoreset=True, next_actions=a, ticks=R)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(T // R):
                eng.launch_step(a, bufs, autoreset=True, next_actions=a, ticks=R)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (5 * T)
        res.append(f"{R:2d}-tick launches {us:6.1f} us/tick ({W * M / us:6.1f} M CASPS)")
    print(f"{name:34s} {eng.launch_shape()} P={eng.tables.scenes[0].num_segments:5d}: " + "; ".join(res))
