"""System identification on the GPU against the reference's
own outputs (tests/golden/sysid.npz): candidate rollouts of every maneuver
kind, and a whole five-stage run_cem whose identified parameters must equal the
reference's exactly (selection only depends on the loss ORDER; the float
losses agree to ~1e-14, CUDA vs libm sin/cos being the only difference)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from cases import GOLDEN
from oracle.sysid import Candidates, rollout
from paper_2605_08528_b200 import sysid as S
from paper_2605_08528_b200.params import VehicleParams

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-9, 1e-9


@pytest.fixture(scope="module")
def g():
    d = np.load(GOLDEN / "sysid.npz")
    return d, json.loads(bytes(d["meta_json"]).decode())


def test_rollouts_match_reference_and_oracle(g, device):
    d, meta = g
    by_id = {m.id: m for m in S.generate_maneuvers(1.0)}
    picked = [by_id[i] for i in meta["picked"]]
    base = VehicleParams()
    got = S.rollout_many(S.ParamBatch(base, d["vectors"]), picked, device)
    for i, (m, ch) in enumerate(zip(picked, got)):
        ora = rollout(Candidates(base, d["vectors"]), m)
        for k in S.CHANNELS:
            assert ch[k].shape == d[f"m{i}_{k}"].shape
            np.testing.assert_allclose(ch[k], d[f"m{i}_{k}"], rtol=RTOL, atol=ATOL, err_msg=f"{m.id} {k}")
            np.testing.assert_allclose(ch[k], ora[k], rtol=RTOL, atol=ATOL, err_msg=f"{m.id} {k} oracle")
    # every candidate x every maneuver of the full set in one launch
    full = S.generate_maneuvers(0.2)
    many = S.rollout_many(S.ParamBatch(base, d["vectors"][:3]), full, device)
    one = S.rollout_channels(S.ParamBatch(base, d["vectors"][:3]), full[5], device)
    for k in S.CHANNELS:
        assert np.array_equal(many[5][k], one[k])


def test_run_cem_matches_reference(g, device):
    d, meta = g
    a = meta["run_cem_args"]
    teacher = S.params_from_vector(d["teacher"], VehicleParams())
    res = S.run_cem(teacher, S.CEMConfig(population=a["population"], total_trials=a["total_trials"]),
                    scale=a["scale"], seed=a["seed"], device=device).to_dict()
    want = meta["run_cem"]
    assert res["trial_split"] == want["trial_split"]
    assert res["best_params"] == want["best_params"]            # identical floats
    for gs, ws in zip(res["stages"], want["stages"]):
        assert (gs["stage"], gs["maneuvers"], gs["trials"]) == (ws["stage"], ws["maneuvers"], ws["trials"])
        assert gs["params"] == ws["params"]
        np.testing.assert_allclose(gs["history"], ws["history"], rtol=RTOL)
        np.testing.assert_allclose(gs["best_loss"], ws["best_loss"], rtol=RTOL)


# ---- the reference's sysid unit contract (pkg/tests/test_sysid.py:55-172), GPU rollouts
def _solo(maneuver, device):
    base = VehicleParams()
    return S.rollout_channels(S.ParamBatch(base, S.params_to_vector(base)[None]), maneuver, device=device)


def test_loss_examples_and_60hz_recording(device):
    m = S.generate_maneuvers(0.07)[0]
    log = _solo(m, device)
    assert log["x"].shape[0] == int(round(m.duration * 60.0))
    assert float(S.sysid_loss(log, log)[0]) == 0.0
    for ch, offset, want in (("x", 1.0, 2.5), ("yaw", 1.0, 0.4)):   # 1.0 MSE + 1.5 terminal; 0.4 weight
        moved = {k: v.copy() for k, v in log.items()}
        moved[ch] = moved[ch] + offset
        assert abs(float(S.sysid_loss(moved, log)[0]) - want) < 1e-12


def test_candidates_are_independent(device):
    base = VehicleParams()
    vecs = np.stack([S.params_to_vector(base)] * 3)
    vecs[1, 0] *= 1.2                                   # more drive torque
    log = S.rollout_channels(S.ParamBatch(base, vecs), S.generate_maneuvers(0.07)[0], device=device)
    assert log["x"].shape[1] == 3
    assert log["x"][-1, 1] > log["x"][-1, 0] and log["x"][-1, 0] == log["x"][-1, 2]


def test_stages_inherit_and_histories_fall(device):
    base = VehicleParams()
    import dataclasses
    teacher = dataclasses.replace(base, tau_drive_max=base.tau_drive_max * 1.1)
    res = S.run_cem(teacher, S.CEMConfig(total_trials=120), base=base, scale=0.05, seed=4, device=device)
    assert res.trial_split == S.allocate_trials(120, S.CEMConfig().stage_weights)
    for st in res.stages:
        h = st["history"]
        assert all(h[i] >= h[i + 1] - 1e-15 for i in range(len(h) - 1))
    s1, s2 = res.stages[0], res.stages[1]
    assert all(k in s1["params"] and k not in s2["params"] for k in ("tau_drive_max", "tau_brake_front"))
    d = res.to_dict()
    assert set(d) == {"trial_split", "stages", "best_params"} and set(d["best_params"]) == set(S.TUNABLE_PARAMS)
