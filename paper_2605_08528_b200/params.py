"""Scalar configuration of the batched vehicle step.

Every field mirrors a dataclass of the reference package (``drivegrid``) so a
config that builds a reference engine builds this one too.  The values are
packed by value into the kernel parameter block (``DgParams`` in
``include/drivegrid_b200.h``); nothing here runs per step.

Reference anchors (``/root/reference/pkg/src/drivegrid``):
  * ``SimConfig``      engine.py:41-67
  * ``ObsConfig``      observation.py:18-35
  * ``RewardConfig``   rewards.py:37-63
  * ``VehicleParams``  vehicle.py:31-84,  ``BicycleParams`` vehicle.py:199-205
  * constants          vehicle.py:20-26, engine.py:31, rewards.py:19-34
"""

from __future__ import annotations

import math
from dataclasses import dataclass, fields
from pathlib import Path

GRAVITY = 9.81
PHYSICS_DT = 1.0 / 120.0
CONTROL_DT = 1.0 / 30.0
DECIMATION = 4
WHEEL_SPEED_LATCH_EPS = 1e-4
WHEEL_SPEED_LIMIT = 200.0
SLIP_SPEED_FLOOR = 0.5
BICYCLE_STEER_MAX = math.radians(30.0)  # == np.deg2rad(30.0) bit for bit
OFFSTAGE_X = 1000.0
CRASH_SPEED_LIMIT = 100.0
TAU_MAX = 10.0

# termination reasons (int8 in the engine, rewards.py:19-24)
REASON_NONE = 0
REASON_GOAL = 1
REASON_COLLISION = 2
REASON_CRASH = 3
REASON_LANE_FORBIDDEN = 4
REASON_TIMEOUT = 5
REASON_NAMES = {0: "none", 1: "goal", 2: "collision", 3: "crash",
                4: "lane_forbidden", 5: "timeout"}

# event order in every (.., 4) event tensor of this package
EVENT_TYPES = ("goal", "collision", "crash", "lane_forbidden")
DENSE_TERMS = ("progress", "lane", "offroad", "idle", "ttc_vehicle", "ttc_edge")
STATE_FIELDS = ("x", "y", "yaw", "v_x", "v_y", "yaw_rate", "steer_angle",
                "steer_rate", "wheel_front", "wheel_rear",
                "brake_sign_front", "brake_sign_rear")
PHASES = ("action", "physics", "observation", "reward_termination", "reset")

LANE_CENTER_CODES = (1, 2)
ROAD_EDGE_CODES = (15, 16)


@dataclass(frozen=True)
class SimConfig:
    num_envs: int = 256
    num_agents: int = 16
    dynamics_mode: str = "dynamic"
    physics_dt: float = PHYSICS_DT
    decimation: int = DECIMATION
    episode_len: int = 1500
    seed: int = 42
    invincible: bool = False
    bbox_half: float = 100.0
    goal_radius: float = 3.0
    num_workers: int = 0

    def __post_init__(self):
        if self.num_agents < 1 or self.num_agents > 16:
            raise ValueError("num_agents must lie in [1, 16]")
        if self.dynamics_mode not in ("dynamic", "bicycle"):
            raise ValueError(f"unknown dynamics_mode {self.dynamics_mode!r}")

    @property
    def control_dt(self) -> float:
        return self.physics_dt * self.decimation

    @property
    def effective_workers(self) -> int:
        return max(1, self.num_workers)


@dataclass(frozen=True)
class ObsConfig:
    k_road: int = 350
    road_radius: float = 10.0
    k_vehicles: int = 24
    ttc_max: float = TAU_MAX
    bbox_half: float = 100.0
    speed_norm: float = 10.0
    type_norm: float = 20.0
    include_weather: bool = True

    @property
    def ego_dim(self) -> int:
        return 7 + (4 if self.include_weather else 0)

    @property
    def obs_dim(self) -> int:
        return self.ego_dim + self.k_road * 5 + self.k_vehicles * 7


@dataclass(frozen=True)
class RewardConfig:
    goal_weight: float = 45.0
    goal_radius: float = 3.0
    collision_weight: float = 6.0
    collision_warmup_steps: int = 24
    crash_weight: float = 10.0
    crash_drift_limit: float = 100.0
    lane_forbidden_weight: float = 20.0
    progress_weight: float = 2.0
    progress_clamp: float = 2.0
    lane_weight: float = 0.08
    lane_sigma: float = 1.75
    lane_heading_weight: float = 0.8
    offroad_weight: float = 0.5
    offroad_lat_limit: float = 3.25
    offroad_dist_limit: float = 6.0
    idle_weight: float = 0.05
    idle_speed: float = 1.0
    ttc_vehicle_alpha: float = 0.10
    ttc_vehicle_pmax: float = 0.35
    ttc_edge_alpha: float = 0.07
    ttc_edge_pmax: float = 0.40
    ttc_floor: float = 0.5
    edge_range: float = 40.0


@dataclass(frozen=True)
class VehicleParams:
    theta_max: float = 0.450
    kp_steer: float = 1839.5
    kd_steer: float = 110.5
    tau_steer_max: float = 1200.0
    tau_drive_max: float = 600.7
    tau_brake_front: float = 1090.5
    tau_brake_rear: float = 980.7
    wheel_mass: float = 37.5
    inertia_scale: float = 1.094
    susp_stiffness: float = 1080.8
    susp_damping: float = 2764.3
    lambda_yaw: float = 10.6
    lambda_lat: float = 150.0
    com_offset: float = 0.0
    f_lon_dry: float = 1.0
    f_lat_dry: float = 1.0
    f_lon_wet: float = 1.0
    f_lat_wet: float = 1.0
    f_lon_gravel: float = 1.0
    f_lat_gravel: float = 1.0
    chassis_mass: float = 1800.0
    wheelbase: float = 2.6
    wheel_radius: float = 0.35
    yaw_inertia: float = 3000.0
    steer_inertia: float = 5.0
    cornering_stiffness: float = 60000.0

    def __post_init__(self):
        for name in ("kp_steer", "kd_steer", "tau_steer_max", "tau_drive_max",
                     "tau_brake_front", "tau_brake_rear"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if not 0.0 < self.theta_max < math.pi / 2:
            raise ValueError("theta_max must lie in (0, pi/2)")

    @property
    def wheel_inertia(self) -> float:
        # same expression order as vehicle.py:79 (left-to-right products)
        return self.inertia_scale * 0.5 * self.wheel_mass * self.wheel_radius ** 2


@dataclass(frozen=True)
class BicycleParams:
    a_max: float = 0.95
    b_max: float = 3.3
    c_roll: float = 0.05


def load_params(path) -> VehicleParams:
    """``name = value`` lines; blank lines and ``#`` comments skipped, later
    keys win (vehicle.py:112-121)."""
    lines = (ln.strip() for ln in Path(path).read_text(encoding="utf-8").splitlines())
    pairs = (ln.partition("=") for ln in lines if ln and not ln.startswith("#"))
    return VehicleParams(**{key.strip(): float(value) for key, _, value in pairs})


def save_params(p: VehicleParams, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(f"{f.name} = {getattr(p, f.name)!r}" for f in fields(p)) + "\n")

