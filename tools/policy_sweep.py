"""Time the policy forward (1024 x 16, actor + critic) for encoder variants
built with -DDG_ENC_AGENTS=<n> (argv), each into its own .so."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_08528_b200 import _native as N  # noqa: E402

variant = sys.argv[1]
lib = Path(f"/tmp/libdg_{variant}.so")
subprocess.run(["/usr/local/cuda/bin/nvcc", *N.NVCC_FLAGS, f"-DDG_ENC_AGENTS={variant}", "-I",
                str(ROOT / "include"), "-o", str(lib), *map(str, N.SOURCES)], check=True,
               capture_output=True)
N.LIB_PATH = lib
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402
from paper_2605_08528_b200.policy import PolicyMLP  # noqa: E402

dev = torch.device("cuda:0")
cfg = C.RootConfig()
cfg.env.num_envs = 1024
eng = Engine(**C.build_inputs(cfg).as_kwargs(), device=dev)
acts = torch.zeros((1024, 16, 3), dtype=torch.float64, device=dev)
obs = eng.observe(as_numpy=False, next_actions=acts)
for _ in range(8):
    obs = eng.step(acts.clone()).obs
    eng.lane_follower(obs, out=acts)
obs = obs.contiguous()
pol = PolicyMLP(eng.obs_config, device=dev, head_scale=1.0)
val = torch.empty((1024, 16), dtype=torch.float32, device=dev)
for _ in range(3):
    pol.forward(obs, actions=acts, value=val)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(50):
        pol.forward(obs, actions=acts, value=val)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"DG_ENC_AGENTS={variant}: policy forward {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
