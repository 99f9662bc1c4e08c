"""Locate GPU-vs-oracle observation differences for one parity case."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import case_inputs  # noqa: E402
from oracle import OracleEngine  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

name = sys.argv[1]
spatial = sys.argv[2] == "1" if len(sys.argv) > 2 else True
case = case_inputs(name)
g = Engine(**case.inputs.as_kwargs(), device=torch.device("cuda:0"), spatial_index=spatial)
o = OracleEngine(**case.inputs.as_kwargs())
go, oo = g.observe(), o.observe()
oc = o.obs_config
bad = np.argwhere(np.abs(go - oo) > 1e-6)
print("n bad", len(bad))
from collections import Counter
print("worlds", Counter(bad[:, 0].tolist()))
print("agents", Counter(bad[:, 1].tolist()))
reg = ["ego" if j < oc.ego_dim else "road" if j < oc.ego_dim + 5 * oc.k_road else "veh" for j in bad[:, 2]]
print("regions", Counter(reg))
print("scene of bad worlds", {int(w): int(case.inputs.assignment[w]) for w in set(bad[:, 0].tolist())})
print("all assignment", case.inputs.assignment.tolist())
for w, m, j in bad[:12]:
    print(w, m, j, go[w, m, j], oo[w, m, j])
