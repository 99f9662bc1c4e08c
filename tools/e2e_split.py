"""Reference-facing numpy loop (bench e2e: 256 x 16, LaneFollower + autoreset)
split into the policy call and the Engine.step call (host wall clock).

  python tools/e2e_split.py [steps]   -> one JSON object
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import os  # noqa: E402

from paper_2605_08528_b200 import _native as N  # noqa: E402

if os.environ.get("DG_LIB_PATH"):          # a variant build
    N.LIB_PATH = Path(os.environ["DG_LIB_PATH"])
    N.load_library(build_if_missing=False)
from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402
from paper_2605_08528_b200.policies import LaneFollower  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
dev = torch.device("cuda:0")
mode = os.environ.get("DG_E2E_MODE")
eng = Engine(**C.build_inputs(C.RootConfig()).as_kwargs(), device=dev,
             launch_mode=None if mode is None else int(mode))
pol = LaneFollower(obs_config=eng.obs_config)
obs = eng.observe()
for _ in range(5):
    obs = eng.step(pol(obs), autoreset=True).obs
torch.cuda.synchronize()
t_pol = t_step = 0.0
t_all = time.perf_counter()
for _ in range(steps):
    t0 = time.perf_counter()
    a = pol(obs)
    t1 = time.perf_counter()
    obs = eng.step(a, autoreset=True).obs
    t2 = time.perf_counter()
    t_pol += t1 - t0
    t_step += t2 - t1
wall = time.perf_counter() - t_all
print(json.dumps({"workload": "256x16 default pool, LaneFollower + autoreset, numpy API", "steps": steps,
                  "ms_per_step": 1e3 * wall / steps, "policy_ms": 1e3 * t_pol / steps,
                  "engine_step_ms": 1e3 * t_step / steps,
                  "casps": eng.W * eng.M * steps / wall, "launch_shape": eng.launch_shape()}))
