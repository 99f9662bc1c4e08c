"""Policy forward (BASELINE configs[4] shape: 1024 x 16 rows, actor + critic)
timed in a CUDA graph, with the valid-slot counts from the step's prefix
record and with the encoder's own scan (outputs must agree bit for bit)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402

import torch  # noqa: E402

from paper_2605_08528_b200 import _native as N  # noqa: E402

if os.environ.get("DG_LIB_PATH"):          # a variant build (tools/policy_variants.py)
    N.LIB_PATH = Path(os.environ["DG_LIB_PATH"])
    N.load_library(build_if_missing=False)

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402
from paper_2605_08528_b200.policy import PolicyMLP  # noqa: E402

dev = torch.device("cuda:0")
cfg = C.RootConfig()
cfg.env.num_envs = 1024
eng = Engine(**C.build_inputs(cfg, device=dev).as_kwargs(), device=dev)
rb = eng.new_rollout_buffers(2)
acts = torch.zeros((1024, 16, 3), dtype=torch.float64, device=dev)
eng.observe(out=rb.obs[1], as_numpy=False, next_actions=acts)
for t in range(8):
    eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=1, ring_start=t % 2)
obs, pre = rb.obs[1].contiguous(), rb.prefix[1].contiguous()
pol = PolicyMLP(eng.obs_config, device=dev, head_scale=1.0)
out = {}
for name, pfx in (("scan", None), ("prefix", pre)):
    a = torch.zeros_like(acts)
    val = torch.empty((1024, 16), dtype=torch.float32, device=dev)
    for _ in range(3):
        pol.forward(obs, actions=a, value=val, prefix=pfx)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            pol.forward(obs, actions=a, value=val, prefix=pfx)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    out[name] = (a.clone(), val.clone())
    print(f"policy forward ({name} counts): {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
print("prefix == scan:", torch.equal(out["scan"][0], out["prefix"][0]) and torch.equal(out["scan"][1], out["prefix"][1]))
