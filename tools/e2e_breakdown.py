"""Where the reference-facing numpy step's time goes (256x16): pinned D2H
bandwidth, the full Engine.step(numpy), the host LaneFollower."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402
from paper_2605_08528_b200.policies import LaneFollower  # noqa: E402

dev = torch.device("cuda:0")
eng = Engine(**C.build_inputs(C.RootConfig()).as_kwargs(), device=dev)
src = torch.empty((256, 16, 1929), dtype=torch.float32, device=dev)
dst = torch.empty(src.shape, dtype=torch.float32, pin_memory=True)
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 20
print(f"D2H 32.3 MB pinned: {dt * 1e3:.3f} ms = {src.numel() * 4 / dt / 1e9:.1f} GB/s")
pol = LaneFollower(obs_config=eng.obs_config)
obs = eng.observe()
for _ in range(3):
    obs = eng.step(pol(obs), autoreset=True).obs
t_pol = t_step = 0.0
for _ in range(30):
    a = time.perf_counter()
    act = pol(obs)
    b = time.perf_counter()
    obs = eng.step(act, autoreset=True).obs
    c = time.perf_counter()
    t_pol += b - a
    t_step += c - b
print(f"LaneFollower(numpy) {t_pol / 30 * 1e3:.3f} ms, Engine.step(numpy) {t_step / 30 * 1e3:.3f} ms, "
      f"phases {dict((k, round(v * 1e3 / 33, 3)) for k, v in eng.phase_seconds.items())}")
