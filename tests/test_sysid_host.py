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


# ---- the reference's sysid unit contract (pkg/tests/test_sysid.py:12-186), host side
def test_desk_scale_keeps_every_tier_and_throttle_brake_coverage():
    man = S.generate_maneuvers(0.07)
    assert all(1 <= v <= 5 for v in S.tier_counts(man).values())
    lon = {m.kind for m in man if m.tier == "longitudinal"}
    assert {"throttle_step", "brake_sweep"} <= lon
    assert [m.id for m in S.generate_maneuvers(0.2)] == [m.id for m in S.generate_maneuvers(0.2)]


def test_schedules_stay_in_the_action_box_and_surface_thirds():
    for m in S.generate_maneuvers(0.3):
        for t in np.linspace(0.0, m.duration, 25):
            a = m.action_at(float(t))
            assert 0.0 <= a[0] <= 1.0 and -1.0 <= a[1] <= 1.0 and 0.0 <= a[2] <= 1.0
    (surf,) = [m for m in S.generate_maneuvers(0.07) if m.tier == "surface"]
    assert [surf.surface_at(t) for t in (0.0, surf.duration / 2, surf.duration - 0.1)] == ["dry", "wet", "gravel"]


def test_cem_settings_validation_and_stages():
    c = S.CEMConfig()
    assert (c.population, c.elite_frac, c.init_std_frac, c.min_std_frac) == (24, 0.25, 0.25, 0.05)
    assert (c.stage_weights, c.refine_window, c.brake_window) == ((0.30, 0.20, 0.15, 0.20, 0.15), 0.18, 0.10)
    for bad in (dict(stage_weights=(0.5, 0.5, 0.1, 0.1, 0.1)), dict(population=2)):
        with pytest.raises(ValueError):
            S.CEMConfig(**bad)
    assert [s.name for s in S.STAGES] == ["longitudinal", "steering", "surface", "refinement", "brake_preservation"]
    assert S.STAGES[3].param_names == S.TUNABLE_PARAMS and S.STAGES[4].param_names == S.LONGITUDINAL_PARAMS


def test_cem_scores_the_incumbent_first_and_ranks_nan_last():
    seen = []

    def f(x):
        seen.append(x.copy())
        return (x ** 2).sum(axis=1)

    start = np.array([0.5, 0.5])
    S.cem_minimize(f, start, -np.ones(2), np.ones(2), trials=8, cfg=S.CEMConfig(population=8),
                   rng=np.random.Generator(np.random.Philox(2)))
    assert np.array_equal(seen[0][0], start)

    def g(x):
        out = (x ** 2).sum(axis=1)
        out[0] = np.nan
        return out

    _, loss, _ = S.cem_minimize(g, np.array([0.5]), np.array([-1.0]), np.array([1.0]), trials=8,
                                cfg=S.CEMConfig(population=8), rng=np.random.Generator(np.random.Philox(3)))
    assert np.isfinite(loss)


def test_param_batch_exposes_candidate_columns():
    base = VehicleParams()
    vecs = np.stack([S.params_to_vector(base)] * 3)
    vecs[1, 0] *= 1.2
    b = S.ParamBatch(base, vecs)
    assert b.batch_size == 3 and b.tau_drive_max.shape == (3,) and b.tau_drive_max[1] == vecs[1, 0]
