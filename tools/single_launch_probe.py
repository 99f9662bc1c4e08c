"""Where a single timed 20-tick launch (the driver's `bench.py --steps 20`)
spends its time beyond 20 x the steady per-tick cost: one-launch graphs
replayed after a sync, repeated; plain launches; back-to-back launches."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

dev = torch.device("cuda:0")
cfg = C.RootConfig()
eng = Engine(**C.build_inputs(cfg, device=dev).as_kwargs(), device=dev)
W, M, D = eng.W, eng.M, eng.obs_config.obs_dim
ring = 9
rb = eng.new_rollout_buffers(ring)
acts = torch.zeros((W, M, 3), dtype=torch.float64, device=dev)
eng.observe(out=rb.obs[ring - 1], as_numpy=False, next_actions=acts)
tick = [0]


def run(R, k=1):
    for _ in range(k):
        eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=R, ring_start=tick[0] % ring)
        tick[0] += R


def ev():
    return torch.cuda.Event(enable_timing=True)


run(20, 3)
for R in (1, 2, 5, 20, 64):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run(R)
    out = []
    for i in range(5):
        torch.cuda.synchronize()
        time.sleep(0.01)
        a, b = ev(), ev()
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    print(f"1-launch graph R={R:3d}: " + " ".join(f"{x:7.1f}" for x in out) + " us")
# no sleep: back-to-back sync'ed replays
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run(20)
out = []
for i in range(5):
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    out.append(a.elapsed_time(b) * 1e3)
print("1-launch graph R=20, no sleep: " + " ".join(f"{x:7.1f}" for x in out) + " us")
out = []
for i in range(5):
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    run(20)
    b.record()
    torch.cuda.synchronize()
    out.append(a.elapsed_time(b) * 1e3)
print("plain launch R=20: " + " ".join(f"{x:7.1f}" for x in out) + " us")
# back-to-back in one graph
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run(20, 10)
torch.cuda.synchronize()
a, b = ev(), ev()
a.record()
g.replay()
b.record()
torch.cuda.synchronize()
print(f"10 x R=20 in one graph: {a.elapsed_time(b) * 1e3 / 10:7.1f} us per launch")
