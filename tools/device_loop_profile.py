"""Host cost of the device-resident closed loop (casps._device_loop: torch CUDA
actions through Engine.step) vs the numpy loop at W x 16, under cProfile.

  python tools/device_loop_profile.py [W] [steps]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import casps  # noqa: E402
from paper_2605_08528_b200.policies import LaneFollower  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
eng = casps._bench_engine(W, 16, "dynamic", 42, torch.device("cuda:0"))
pol = LaneFollower(obs_config=eng.obs_config)
for name, loop in (("vectorized", casps._host_loop), ("device", casps._device_loop)):
    loop(eng, pol, 10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loop(eng, pol, steps)
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / steps * 1e6:.1f} us/step")
pr = cProfile.Profile()
pr.enable()
casps._device_loop(eng, pol, steps)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
