"""Configuration surface (no GPU): the behaviours the reference's own config
tests pin (pkg/tests/test_config_cli.py:19-101) -- defaults from an empty
file, unknown keys rejected with their dotted path, YAML round trip, every
reward weight reachable, weather / goal draws deterministic -- restated
against this package's config.py / goals.py."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.goals import polyline_arc_point, resample_goal
from paper_2605_08528_b200.params import RewardConfig, SimConfig
from paper_2605_08528_b200.scenes import prepare_scene, straight_scene


def test_empty_and_missing_documents_give_defaults(tmp_path):
    f = tmp_path / "empty.yaml"
    f.write_text("")
    for cfg in (C.parse_config(f), C.parse_config(None), C.config_from_dict(None)):
        assert (cfg.env.num_envs, cfg.env.num_agents_per_env, cfg.env.episode_len) == (256, 16, 1500)
        assert cfg.env.dynamics_mode == "dynamic" and cfg.seed == 42


def test_non_mapping_root_and_unknown_keys_rejected(tmp_path):
    f = tmp_path / "list.yaml"
    f.write_text("- 1\n- 2\n")
    with pytest.raises(C.ConfigError, match="mapping"):
        C.parse_config(f)
    with pytest.raises(C.ConfigError, match=r"weather\.wet_frac$"):
        C.config_from_dict({"weather": {"wet_frac": 0.5}})
    with pytest.raises(C.ConfigError, match="obss"):
        C.config_from_dict({"obss": {}})
    assert issubclass(C.ConfigError, ValueError)


def test_yaml_round_trip(tmp_path):
    cfg = C.RootConfig()
    cfg.env.num_envs, cfg.seed = 24, 3
    cfg.weather.wet_fraction = 0.4
    cfg.eval.random_goals = True
    cfg.reward = dataclasses.replace(cfg.reward, collision_weight=-9.0)
    f = tmp_path / "round.yaml"
    C.save_config(cfg, f)
    assert C.config_to_dict(C.parse_config(f)) == C.config_to_dict(cfg)


def test_every_reward_weight_reachable_from_yaml():
    for fld in dataclasses.fields(RewardConfig):
        probe = 3 if fld.type in ("int", int) else 3.5
        assert getattr(C.config_from_dict({"reward": {fld.name: probe}}).reward, fld.name) == probe


def test_weather_draws_deterministic_and_in_range():
    w = C.WeatherConfig(wet_fraction=0.5)
    a, b = C.sample_weather(w, 32, seed=9), C.sample_weather(w, 32, seed=9)
    assert a == b
    films = [h for _, h in a]
    assert any(h > 0 for h in films) and any(h == 0 for h in films)
    assert all(s in ("AC", "SMA", "OGFC") for s, _ in a)
    assert all(0.0 <= h <= w.film_max_mm for h in films)


def _straight():
    scene = prepare_scene(straight_scene(agent_count=1))
    return scene, np.asarray(scene.agents[0].start, dtype=np.float64)


def test_goal_at_fixed_distance_lies_that_far_along_the_lane():
    scene, start = _straight()
    goal = resample_goal(start, scene, 20.0, 20.0, np.random.Generator(np.random.Philox(0)))
    assert goal is not None and abs(np.hypot(*(goal - start)) - 20.0) < 1e-9


def test_goal_beyond_the_lane_is_none_and_draws_repeat():
    scene, start = _straight()
    assert resample_goal(start, scene, 1e5, 1e5, np.random.Generator(np.random.Philox(0))) is None
    a = resample_goal(start, scene, 10.0, 60.0, np.random.Generator(np.random.Philox(5)))
    b = resample_goal(start, scene, 10.0, 60.0, np.random.Generator(np.random.Philox(5)))
    assert np.array_equal(a, b)


def test_polyline_arc_point_ends_and_interpolation():
    pts = np.array([[0.0, 0.0], [3.0, 4.0], [3.0, 10.0]])     # arc lengths 0, 5, 11
    assert np.array_equal(polyline_arc_point(pts, 0.0, 0.0), [0.0, 0.0])
    assert np.array_equal(polyline_arc_point(pts, 0.0, 11.0), [3.0, 10.0])
    assert np.allclose(polyline_arc_point(pts, 5.0, 3.0), [3.0, 7.0])
    assert np.allclose(polyline_arc_point(pts, 5.0, -2.5), [1.5, 2.0])
    assert polyline_arc_point(pts, 0.0, 11.5) is None and polyline_arc_point(pts, 5.0, -5.5) is None


def test_sim_config_checks():
    cfg = SimConfig(num_envs=2, num_agents=4)
    assert abs(cfg.control_dt - 1 / 30) < 1e-15 and abs(cfg.episode_len * cfg.control_dt - 50.0) < 1e-9
    for bad in (dict(num_agents=17), dict(dynamics_mode="warp")):
        with pytest.raises(ValueError):
            SimConfig(**bad)


def test_vehicle_params_file_round_trip_and_config_path(tmp_path):
    """save_params / load_params (vehicle.py:105-121) and
    ``vehicle_params_path`` in the YAML config."""
    from paper_2605_08528_b200.params import VehicleParams, load_params, save_params
    p = dataclasses.replace(VehicleParams(), tau_drive_max=1234.5, com_offset=-0.125)
    f = tmp_path / "veh.txt"
    save_params(p, f)
    assert load_params(f) == p
    f.write_text("# tuned\n\ntau_drive_max = 999.0\nkp_steer=10\n")
    q = load_params(f)
    assert q.tau_drive_max == 999.0 and q.kp_steer == 10.0 and q.wheel_mass == VehicleParams().wheel_mass
    cfg = C.config_from_dict({"vehicle_params_path": str(f), "env": {"num_envs": 2, "num_agents_per_env": 2}})
    assert C.build_inputs(cfg).params == q
