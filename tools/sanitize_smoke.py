"""A small pass over every kernel (step fused / split / persistent rollout,
observe, reset, LaneFollower, DRAC, sysid, policy forward + sampling, GAE),
sized for compute-sanitizer runs (tools/gpu_sanitize.sh)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import cfg_of  # noqa: E402
from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200 import metrics as GM  # noqa: E402
from paper_2605_08528_b200 import sysid as S  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402
from paper_2605_08528_b200.params import VehicleParams  # noqa: E402
from paper_2605_08528_b200.policy import PolicyMLP, gae  # noqa: E402

dev = torch.device("cuda:0")
inp = C.build_inputs(cfg_of(4, 16, seed=31))
acts = np.random.Generator(np.random.Philox(0)).uniform(-1, 1, (4, 4, 16, 3))
for mode in (0, 1):
    e = Engine(**inp.as_kwargs(), device=dev, launch_mode=mode)
    e.track_episode_metrics()
    for t in range(3):
        e.step(acts[t], autoreset=True)
    e.teleport_reset(np.ones((4, 16), bool))
    e.episode_metrics()
e = Engine(**inp.as_kwargs(), device=dev)
out = e.rollout(torch.as_tensor(acts, device=dev), autoreset=True)
a = torch.zeros((4, 16, 3), dtype=torch.float64, device=dev)
e.rollout(a, ticks=3, policy="lane_follower")
pol = PolicyMLP(device=dev)
v = torch.empty((3, 4, 16), dtype=torch.float32, device=dev)
lp = torch.empty_like(v)
r = e.rollout(a, ticks=3, policy=pol, values=v, sample=True, log_probs=lp)
gae(r.rewards[1:], r.dones[1:], v)
st = {k: np.zeros((2, 4, 16)) for k in ("x", "y", "yaw", "v_x", "v_y")}
GM.episode_metrics([{"state": {k: st[k][i] for k in st}, "alive_pre": np.ones((4, 16), bool),
                     "events": {"goal": np.zeros((4, 16), bool), "collision": np.zeros((4, 16), bool)}}
                    for i in range(2)], np.ones((4, 16), bool))
S.rollout_many(S.ParamBatch(VehicleParams(), S.params_to_vector(VehicleParams())[None].repeat(3, 0)),
               S.generate_maneuvers(0.1)[:2])
# round 2: on-device world construction (+ random goals, padded batch, subsets),
# mode 2 with the pipelined tail on a resident ring over multi-tick launches,
# the fused global-geometry variants, the policy encoder's work queue
from paper_2605_08528_b200.scenes import prepare_scene, straight_scene  # noqa: E402

cfg = cfg_of(6, 16, seed=5)
cfg.eval.random_goals, cfg.eval.goal_min_m, cfg.eval.goal_max_m = True, 10.0, 40.0
e = C.build_engine(cfg, device=dev)
_ = (e.worlds.midpoints, e.lane, e.edge)
rb = e.new_rollout_buffers(3)
a = torch.zeros((6, 16, 3), dtype=torch.float64, device=dev)
e.observe(out=rb.obs[2], as_numpy=False, next_actions=a)
for k in range(3):
    e.launch_step(a, rb, autoreset=True, next_actions=a, ticks=4, ring_start=(4 * k) % 3)
lanes = tuple(float(x) for x in np.round(np.arange(-9.0, 9.01, 0.25), 2))
dense = prepare_scene(straight_scene("dense", lane_offsets=lanes, agent_count=4, agent_gap=15.0, goal_dist=40.0))
for mode in (0, 2):
    g = Engine(**C.build_inputs(cfg_of(2, 4, seed=3), scenes=[dense]).as_kwargs(), device=dev, launch_mode=mode)
    a2 = g.lane_follower(g.observe_device())
    g.rollout(a2, ticks=3, policy="lane_follower", autoreset=True)
e.run_mlp_ticks(a, rb, pol, 2, autoreset=True, values=torch.empty((2, 6, 16), dtype=torch.float32, device=dev))
torch.cuda.synchronize()
print("sanitize smoke done")
