"""``drivegrid_bindings`` drop-in on the GPU: the handle contract of the
reference's binding tests (pkg/bindings/tests/test_bindings.py:37-132) --
default shapes, missing config file, bicycle mode, deterministic float32
resets, shape validation, zero reward after termination, a replayed action
stream matching the engine (and the oracle) element for element -- restated
against this package's make_env / EnvHandle."""

from __future__ import annotations

import json

import numpy as np
import pytest
import yaml

from oracle import OracleEngine
from paper_2605_08528_b200 import config as C
from paper_2605_08528_b200.bindings import make_env
from paper_2605_08528_b200.policies import ReplayPolicy

pytestmark = pytest.mark.gpu


def _cfg_file(tmp_path, W=2, M=3, mode="dynamic", seed=11):
    f = tmp_path / "cfg.yaml"
    f.write_text(yaml.safe_dump({"env": {"num_envs": W, "num_agents_per_env": M, "dynamics_mode": mode},
                                 "scene_factory": {"assignment_mode": "fixed"}, "seed": seed}))
    return f


def _action_stream(tmp_path, T, W, M, seed=3):
    acts = np.random.Generator(np.random.Philox(seed)).uniform(-1.0, 1.0, (T, W, M, 3))
    f = tmp_path / "actions.jsonl"
    with open(f, "w") as fh:
        for (t, w, m), a in np.ndenumerate(acts[..., 0]):
            fh.write(json.dumps({"step": t, "world": w, "agent": m, "action": acts[t, w, m].tolist()}) + "\n")
    return f, acts


def test_defaults_and_missing_file(device):
    env = make_env(None, device=device)
    assert env.shapes["obs"] == (256, 16, 1929) and env.shapes["actions"] == (256, 16, 3)
    with pytest.raises(FileNotFoundError):
        make_env("/nonexistent/config.yaml", device=device)


def test_bicycle_mode(device, tmp_path):
    assert make_env(_cfg_file(tmp_path, mode="bicycle"), device=device).reset().shape == (2, 3, 1929)


def test_reset_is_deterministic_float32(device, tmp_path):
    f = _cfg_file(tmp_path)
    env = make_env(f, device=device)
    a = env.reset()
    env.step(np.zeros((2, 3, 3)))
    b, info = env.reset(return_info=True)
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert info["alive"].shape == (2, 3)
    assert np.array_equal(make_env(f, device=device).reset(), a)
    with pytest.raises(ValueError, match="shape"):
        env.step(np.zeros((2, 2, 3)))


def test_terminated_agent_reward_is_zero(device, tmp_path):
    env = make_env(_cfg_file(tmp_path, W=1, M=1), device=device)
    env.reset()
    acts = np.zeros((1, 1, 3))
    acts[..., 0] = 1.0
    finished = False
    for _ in range(1500):
        _, rewards, dones, _ = env.step(acts)
        if finished:
            assert rewards[0, 0] == 0.0
            break
        finished = bool(dones[0, 0])
    assert finished


def test_replayed_stream_matches_engine_and_oracle(device, tmp_path):
    """50 replayed steps (ReplayPolicy.from_jsonl) through the handle equal the
    engine stepped directly, bit for bit, and the oracle within the parity
    tolerances (integer / boolean outputs exact)."""
    W, M, T = 2, 3, 50
    f = _cfg_file(tmp_path, W, M, seed=17)
    stream, acts = _action_stream(tmp_path, T, W, M)
    replay = ReplayPolicy.from_jsonl(stream, W, M)
    assert np.array_equal(replay.actions, acts)
    env = make_env(f, device=device)
    env.reset()
    eng = C.build_engine(C.parse_config(f), device=device)
    ora = OracleEngine(**C.build_inputs(C.parse_config(f)).as_kwargs())
    for t in range(T):
        a = replay(None)
        obs, rew, done, info = env.step(a)
        out = eng.step(a)
        assert np.array_equal(obs, out.obs) and np.array_equal(rew, out.rewards) and np.array_equal(done, out.dones)
        o = ora.step(a)
        assert np.array_equal(done, o.dones) and np.array_equal(info["reason"], o.info["reason"])
        assert np.allclose(rew, o.rewards, rtol=1e-9, atol=1e-9)
        assert np.allclose(obs, o.obs, rtol=1e-6, atol=1e-6)
    assert obs.shape == (W, M, 1929)


def test_cuda_actions_keep_the_step_in_hbm(device, tmp_path):
    """A torch CUDA action batch goes straight to the kernel and every output
    comes back as a CUDA tensor, equal to the numpy round trip of a twin
    handle; a mis-shaped CUDA batch is rejected the same way."""
    import torch
    f = _cfg_file(tmp_path, W=3, M=4, seed=5)
    host, dev = make_env(f, device=device), make_env(f, device=device)
    host.reset()
    dev.reset()
    acts = np.random.Generator(np.random.Philox(8)).uniform(-1.0, 1.0, (10, 3, 4, 3))
    for t in range(10):
        o_h, r_h, d_h, i_h = host.step(acts[t])
        o_d, r_d, d_d, i_d = dev.step(torch.as_tensor(acts[t], device=device))
        assert o_d.is_cuda and r_d.is_cuda and d_d.is_cuda
        assert np.array_equal(o_d.cpu().numpy(), o_h) and np.array_equal(r_d.cpu().numpy(), r_h)
        assert np.array_equal(d_d.cpu().numpy(), d_h)
        assert np.array_equal(i_d["reason"].cpu().numpy(), i_h["reason"])
    with pytest.raises(ValueError, match="shape"):
        dev.step(torch.zeros((3, 5, 3), device=device))
