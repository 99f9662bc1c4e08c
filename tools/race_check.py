"""Repeat observe()/step on identical inputs and report any run-to-run drift."""
import sys
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import case_inputs  # noqa: E402
from oracle import OracleEngine  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

for name in sys.argv[1:]:
    case = case_inputs(name)
    ora = OracleEngine(**case.inputs.as_kwargs()).observe()
    oc = case.inputs.obs
    for trial in range(20):
        g = Engine(**case.inputs.as_kwargs(), device=torch.device("cuda:0"))
        for rep in range(5):
            go = g.observe()
            bad = np.argwhere(np.abs(go - ora) > 1e-6)
            if len(bad):
                reg = Counter("ego" if j < oc.ego_dim else "road" if j < oc.ego_dim + 5 * oc.k_road else "veh"
                              for j in bad[:, 2])
                print(name, "trial", trial, "rep", rep, "nbad", len(bad), dict(reg),
                      "worlds", sorted(Counter(bad[:, 0].tolist()).items())[:6],
                      "agents", sorted(Counter(bad[:, 1].tolist()).items())[:6])
                w, m, j = bad[0]
                print("   first", w, m, j, go[w, m, j], ora[w, m, j], "row nz gpu", (go[w, m] != 0).sum(), "ora", (ora[w, m] != 0).sum())
print("done")
