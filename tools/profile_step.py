"""Small driver for ncu: a few fused steps at a chosen W x 16 (default 256)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = C.RootConfig()
cfg.env.num_envs = W
eng = Engine(**C.build_inputs(cfg).as_kwargs(), device=torch.device("cuda:0"))
acts = torch.zeros((W, 16, 3), dtype=torch.float64, device="cuda:0")
bufs = eng.new_step_buffers()
obs = eng.observe_device()
for i in range(steps):
    eng.lane_follower(bufs.obs if i else obs, out=acts)
    eng.launch_step(acts, bufs, autoreset=True)
torch.cuda.synchronize()
print("done", W, steps)
