"""Oracle pin for the integer decisions (CPU): the oracle's road slot ->
segment map, neighbour order and nearest-lane index equal the reference's own
argsort / argmin results, captured by tests/golden/make_golden.py
(index_pins) from the unmodified reference step."""

from __future__ import annotations

import numpy as np
import pytest

from cases import GOLDEN, cfg_of, event_actions
from oracle import OracleEngine
from paper_2605_08528_b200 import config as C


@pytest.mark.parametrize("name", ["traj_events", "traj_pool"])
def test_oracle_index_record_matches_reference(name):
    g = np.load(GOLDEN / f"{name}_indices.npz")
    cfg = cfg_of(4, 16, seed=31) if name == "traj_events" else cfg_of(4, 16)
    ora = OracleEngine(**C.build_inputs(cfg).as_kwargs(), num_workers=1)
    ora.record_indices = True
    steps = g["lane"].shape[0]
    acts = g["actions"]
    if name == "traj_events":
        assert np.array_equal(acts, event_actions(steps, 4, 16).astype(np.float64))
    checked_lanes = 0
    for t in range(steps):
        rec = ora.step(acts[t]).info["indices"]
        assert np.array_equal(rec.lane, g["lane"][t]), f"step {t + 1}: nearest lane"
        assert np.array_equal(rec.road_n, g["road_n"][t]), f"step {t + 1}: road count"
        assert np.array_equal(rec.veh_n, g["veh_n"][t]), f"step {t + 1}: neighbour count"
        assert np.array_equal(rec.road, g["road"][t]), f"step {t + 1}: road order"
        assert np.array_equal(rec.veh, g["veh"][t]), f"step {t + 1}: neighbour order"
        checked_lanes += int((rec.lane >= 0).sum())
    assert checked_lanes > 0
