"""CPU oracle of the sysid candidate rollouts -- TEST INFRASTRUCTURE ONLY.

Numpy restatement of sysid.py:201-228 (rollout_channels over a ParamBatch)
on top of this oracle's 120 Hz substep (oracle/stepper.py, vehicle.py:237-336)
with the candidate parameters broadcast along the batch axis.  Pinned against
the reference's own rollouts in tests/golden/sysid.npz.
"""

from __future__ import annotations

import numpy as np

from paper_2605_08528_b200 import params as P

from .stepper import decode, substep_dynamic

TUNABLE = ("tau_drive_max", "tau_brake_front", "tau_brake_rear", "theta_max", "kp_steer", "kd_steer",
           "tau_steer_max", "wheel_mass", "inertia_scale", "susp_stiffness", "susp_damping", "lambda_yaw",
           "lambda_lat", "com_offset", "f_lon_dry", "f_lat_dry", "f_lon_wet", "f_lat_wet", "f_lon_gravel",
           "f_lat_gravel")
BASE_MU = {"dry": 1.0, "wet": 0.75, "gravel": 0.60}


class Candidates:
    """Duck-typed VehicleParams whose tunable fields are (B,) arrays (sysid.py:174-198)."""

    def __init__(self, base: P.VehicleParams, vectors):
        v = np.atleast_2d(np.asarray(vectors, dtype=np.float64))
        self.B = v.shape[0]
        for f in P.VehicleParams.__dataclass_fields__:
            setattr(self, f, getattr(base, f))
        for i, name in enumerate(TUNABLE):
            setattr(self, name, v[:, i].copy())

    @property
    def wheel_inertia(self):
        return self.inertia_scale * 0.5 * self.wheel_mass * self.wheel_radius ** 2

    def mu(self, surface):
        return np.minimum(1.0, BASE_MU[surface] * np.sqrt(getattr(self, f"f_lon_{surface}")
                                                          * getattr(self, f"f_lat_{surface}")))


def rollout(cands: Candidates, maneuver) -> dict:
    """(T60, B) channels of one maneuver; ``maneuver`` provides action_at /
    surface_at / duration."""
    B = cands.B
    s = {k: np.zeros(B) for k in P.STATE_FIELDS}
    s["brake_sign_front"] = np.ones(B)
    s["brake_sign_rear"] = np.ones(B)
    rec = {k: [] for k in ("x", "y", "yaw", "speed", "yaw_rate", "wheel_speed", "steer_angle")}
    for tick in range(int(round(maneuver.duration / P.CONTROL_DT))):
        t = tick * P.CONTROL_DT
        act = decode(np.asarray(maneuver.action_at(t), dtype=np.float64))
        mu = cands.mu(maneuver.surface_at(t))
        for sub in range(P.DECIMATION):
            s = substep_dynamic(s, act, mu, cands, P.PHYSICS_DT)
            if sub % 2:
                rec["x"].append(s["x"])
                rec["y"].append(s["y"])
                rec["yaw"].append(s["yaw"])
                rec["speed"].append(np.sqrt(s["v_x"] ** 2 + s["v_y"] ** 2))
                rec["yaw_rate"].append(s["yaw_rate"])
                rec["wheel_speed"].append(0.5 * (s["wheel_front"] + s["wheel_rear"]))
                rec["steer_angle"].append(s["steer_angle"])
    return {k: np.stack(v) for k, v in rec.items()}
