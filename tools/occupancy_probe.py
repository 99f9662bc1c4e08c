"""Launch one bench-shaped step with a given mode-2 shape (argv: warps) --
for ncu's occupancy / launch-stats sections."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

dev = torch.device("cuda:0")
eng = Engine(**C.build_inputs(C.RootConfig(), device=dev).as_kwargs(), device=dev)
eng.tune(int(sys.argv[1]), 0, mode=2)
rb = eng.new_rollout_buffers(2)
acts = torch.zeros((eng.W, eng.M, 3), dtype=torch.float64, device=dev)
eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=4)
torch.cuda.synchronize()
print("smem bytes per CTA:", eng._lib and eng.launch_shape())
