"""Weather / road surface -> per-world friction coefficient (host, init only).

The hot path consumes two per-world values: ``mu_eff`` (the friction-circle
coefficient used by every physics substep) and the 4-wide weather token
appended to the ego observation.  Both are produced here once per engine from
the closed-form steady state of the averaged bristle (LuGre) model with the
frozen hydro-lift fit, exactly as the reference evaluates them.

Reference anchors (``/root/reference/pkg/src/drivegrid/friction.py``):
  * Stribeck speed / g(v)        98-111
  * bristle steady state          114-124
  * hydro lift Y_R / Y_F          161-198 (coefficients: data/hydro_coeffs.json)
  * LuGre default solve           201-235
  * mu_effective                  243-274
  * assign_friction / token       355-382,  ground_material 385-388
Offline calibration (least-squares fit, ODE integration) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

STRIBECK_B = (4.8916, -7.91, 3.01, 3.40)
REFERENCE_SPEED = 13.89
SLIP_STATIC = 0.15
SLIP_DYNAMIC = 0.80
MU_FLOOR = 1e-3
H_NORM_MM = 1.0
AQUAPLANE_CENTER = 0.86
AQUAPLANE_WIDTH = 0.008

# frozen hydro-lift fit shipped with the reference (data/hydro_coeffs.json)
HYDRO_COEFFS = {
    "y_inf": 0.8217611195465648,
    "a": 2.0428206057970026,
    "p": 1.7294371296215756,
    "q": 19.999999999999996,
    "c1": 0.013880289683053907,
    "c2": 0.05000000000000001,
}


@dataclass(frozen=True)
class SurfacePreset:
    name: str
    theta: float
    texture_amplitude_mm: float


SURFACES = {
    "AC": SurfacePreset("AC", 1.00, 0.65),
    "SMA": SurfacePreset("SMA", 1.09, 0.80),
    "OGFC": SurfacePreset("OGFC", 1.21, 1.08),
}
SURFACE_ORDER = ("AC", "SMA", "OGFC")


def surface(name: str) -> SurfacePreset:
    if name not in SURFACES:
        raise ValueError(f"unknown surface {name!r}; expected one of {SURFACE_ORDER}")
    return SURFACES[name]


@dataclass(frozen=True)
class LuGreParams:
    sigma0: float
    mu_s_stribeck: float
    mu_c_stribeck: float
    alpha_stribeck: float = 1.0
    contact_length: float = 0.15

    @property
    def K(self) -> float:
        return 7.0 / (6.0 * self.contact_length)


def stribeck_speed(h_w_m):
    h = np.asarray(h_w_m, dtype=np.float64)
    if (h < 0).any():
        raise ValueError("water film thickness must be non-negative")
    b1, b2, b3, b4 = STRIBECK_B
    out = b1 * np.exp(1000.0 * b2 * h + b3) + b4
    return float(out) if out.ndim == 0 else out


def _stribeck_g(v_r, prm: LuGreParams, v_s):
    return prm.mu_c_stribeck + (prm.mu_s_stribeck - prm.mu_c_stribeck) * np.exp(
        -np.abs(np.asarray(v_r) / v_s) ** prm.alpha_stribeck)


def bristle_steady_state(v_r, w_r, theta, y_r, prm: LuGreParams, h_w_m=0.0):
    """z* = v_r / lambda for dz/dt = v_r - lambda z."""
    g = _stribeck_g(v_r, prm, stribeck_speed(h_w_m))
    lam = theta * y_r * (prm.sigma0 * np.abs(v_r) / g + prm.K * np.abs(w_r))
    return np.asarray(v_r) / lam


@dataclass(frozen=True)
class HydroLiftModel:
    y_inf: float
    a: float
    p: float
    q: float
    c1: float
    c2: float

    def _u(self, v, h_mm):
        return (np.asarray(v, dtype=np.float64) / REFERENCE_SPEED) * np.asarray(h_mm, dtype=np.float64)

    def contact_ratio(self, v, h_mm):
        u = self._u(v, h_mm)
        base = self.y_inf + (1.0 - self.y_inf) * (1.0 + (u / self.a) ** self.p) ** (-self.q)
        gate = 1.0 / (1.0 + np.exp(np.clip((u - AQUAPLANE_CENTER) / AQUAPLANE_WIDTH, -60.0, 60.0)))
        return base * gate

    def lift_ratio(self, v, h_mm):
        u = self._u(v, h_mm)
        return np.minimum(self.c1 * np.maximum(u, 0.0) ** self.c2, 1.0)


@lru_cache(maxsize=1)
def default_hydro_model() -> HydroLiftModel:
    return HydroLiftModel(**HYDRO_COEFFS)


@lru_cache(maxsize=1)
def default_lugre_params(dry_static_mu=1.1048, dynamic_ratio=0.99, contact_length=0.15,
                         alpha=1.0, mu_c_ratio=0.75) -> LuGreParams:
    """Pin (sigma0, mu_s) from the two dry anchors: a 2x2 system linear in
    (1/mu_s, 1/sigma0) (friction.py:201-235)."""
    K = 7.0 / (6.0 * contact_length)
    v_s0 = stribeck_speed(0.0)

    def q_of(slip):
        v_r = slip * REFERENCE_SPEED
        return mu_c_ratio + (1.0 - mu_c_ratio) * np.exp(-((v_r / v_s0) ** alpha))

    A = np.array([
        [1.0 / q_of(SLIP_STATIC), K * (1.0 - SLIP_STATIC) / SLIP_STATIC],
        [1.0 / q_of(SLIP_DYNAMIC), K * (1.0 - SLIP_DYNAMIC) / SLIP_DYNAMIC],
    ])
    rhs = np.array([1.0 / dry_static_mu, 1.0 / (dynamic_ratio * dry_static_mu)])
    inv_mu_s, inv_sigma0 = np.linalg.solve(A, rhs)
    mu_s = 1.0 / inv_mu_s
    return LuGreParams(1.0 / inv_sigma0, mu_s, mu_c_ratio * mu_s, alpha, contact_length)


def mu_effective(surface_name: str, h_mm: float, v=REFERENCE_SPEED, slip=SLIP_STATIC,
                 hydro: HydroLiftModel | None = None, params: LuGreParams | None = None) -> float:
    if v < 0:
        raise ValueError("speed must be non-negative")
    if not 0.0 <= slip <= 1.0:
        raise ValueError("slip ratio must lie in [0, 1]")
    preset = surface(surface_name)
    hydro = hydro or default_hydro_model()
    prm = params or default_lugre_params()
    v_r = slip * v
    w_r = (1.0 - slip) * v
    if v_r == 0.0 and w_r == 0.0:
        return 0.0
    y_r = float(hydro.contact_ratio(v, h_mm))
    y_f = float(hydro.lift_ratio(v, h_mm))
    contact = max(preset.theta * y_r - y_f, 0.0)
    if contact == 0.0 or v_r == 0.0:
        return 0.0
    z_star = bristle_steady_state(v_r, w_r, preset.theta, y_r, prm, h_mm * 1e-3)
    return float(contact * preset.theta * y_r * prm.sigma0 * z_star)


@dataclass(frozen=True)
class FrictionAssignment:
    surface: SurfacePreset
    water_film_mm: float
    mu_static: float
    mu_dynamic: float
    weather_token: np.ndarray  # [h/1mm, 1_AC, 1_SMA, 1_OGFC]


def weather_token(surface_name: str, h_mm: float) -> np.ndarray:
    return np.array([h_mm / H_NORM_MM] + [1.0 if surface_name == n else 0.0 for n in SURFACE_ORDER],
                    dtype=np.float64)


def assign_friction(surface_name: str, h_mm: float, hydro=None, params=None) -> FrictionAssignment:
    mu_s = max(mu_effective(surface_name, h_mm, REFERENCE_SPEED, SLIP_STATIC, hydro, params), MU_FLOOR)
    mu_d = max(mu_effective(surface_name, h_mm, REFERENCE_SPEED, SLIP_DYNAMIC, hydro, params), MU_FLOOR)
    return FrictionAssignment(surface(surface_name), h_mm, mu_s, mu_d,
                              weather_token(surface_name, h_mm))


def ground_material(f_surface: float, f_lon: float, f_lat: float):
    mu_s = min(1.0, f_surface * np.sqrt(f_lon * f_lat))
    return float(mu_s), float(0.95 * mu_s)


def effective_contact_mu(assignment: FrictionAssignment, ground_mu_s: float) -> float:
    return min(assignment.mu_static, ground_mu_s)
