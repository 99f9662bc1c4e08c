"""System identification, host side (no GPU): the maneuver sets, the loss,
the CEM pieces and the CPU oracle's candidate rollouts against the
reference's own outputs (tests/golden/sysid.npz, make_golden.py sysid)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from cases import GOLDEN
from oracle.sysid import Candidates, rollout
from paper_2605_08528_b200 import sysid as S
from paper_2605_08528_b200.params import VehicleParams


@pytest.fixture(scope="module")
def g():
    d = np.load(GOLDEN / "sysid.npz")
    return d, json.loads(bytes(d["meta_json"]).decode())


def test_maneuver_sets_match_reference(g):
    _, meta = g
    for sc, want in meta["maneuvers"].items():
        got = [[m.id, m.tier, m.kind, m.duration, m.params] for m in S.generate_maneuvers(float(sc))]
        assert json.loads(json.dumps(got)) == want, sc
    assert S.tier_counts(S.generate_maneuvers(1.0)) == {"longitudinal": 17, "lateral": 64, "combined": 18,
                                                         "frequency": 39, "surface": 1}


def test_bounds_and_trial_split(g):
    d, _ = g
    lo, hi = S.default_bounds(VehicleParams())
    assert np.array_equal(lo, d["lo"]) and np.array_equal(hi, d["hi"])
    assert S.allocate_trials(320, S.CEMConfig().stage_weights) == [96, 64, 48, 64, 48]


def _picked(meta):
    by_id = {m.id: m for m in S.generate_maneuvers(1.0)}
    return [by_id[i] for i in meta["picked"]]


def test_oracle_rollouts_and_loss_match_reference(g):
    d, meta = g
    base = VehicleParams()
    cands = Candidates(base, d["vectors"])
    teach = Candidates(base, d["teacher"][None, :])
    for i, m in enumerate(_picked(meta)):
        st, te = rollout(cands, m), rollout(teach, m)
        for k in S.CHANNELS:
            assert np.array_equal(st[k], d[f"m{i}_{k}"]), (m.id, k)
            assert np.array_equal(te[k], d[f"m{i}_teacher_{k}"]), (m.id, k)
        assert np.array_equal(S.sysid_loss(st, te), d[f"m{i}_loss"]), m.id


def test_cem_toy_quadratic():
    rng = np.random.Generator(np.random.Philox(0))
    lo, hi = -np.ones(3), np.ones(3)
    x, f, hist = S.cem_minimize(lambda s: ((s - 0.3) ** 2).sum(1), np.zeros(3), lo, hi, 200,
                                S.CEMConfig(population=20), rng)
    assert f < 1e-3 and np.all(np.diff(hist) <= 0) and np.allclose(x, 0.3, atol=0.05)
