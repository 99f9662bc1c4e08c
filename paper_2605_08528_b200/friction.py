"""Weather / road surface -> per-world friction coefficient (host, init only).

The step consumes two per-world values: ``mu_eff`` (the friction-circle
coefficient of every physics substep) and the 4-wide weather token appended
to the ego observation.  They come from the closed-form steady state of the
averaged bristle (LuGre) model with the frozen hydro-lift fit, evaluated here
as ONE array expression over all worlds (``mu_table``): an engine of 65,536
worlds assigns its friction in a fraction of a second instead of a scalar
call per world.  Each float64 operation is the reference's, in its order, so
every value is bit-identical to the reference's scalar evaluation (pinned by
tests/golden/friction.npz and the table-vs-reference test).  One care point:
the reference raises numpy SCALARS to powers, which numpy evaluates with the
C library's pow, while numpy's array power may take a SIMD (SVML) kernel
that differs in the last ulp -- so powers go through ``_pow`` (libm pow per
distinct base); every other operation is the same ufunc either way.

Reference anchors (``/root/reference/pkg/src/drivegrid/friction.py``):
  * Stribeck speed v_s(h), g(v)        98-111
  * bristle steady state z*            114-124
  * hydro lift Y_R (contact), Y_F      161-198 (coefficients: data/hydro_coeffs.json)
  * LuGre default (sigma0, mu_s) solve 201-235
  * mu_effective                       243-274
  * assign_friction / weather token    355-382,  ground_material 385-388
Offline calibration (least-squares fit, ODE integration) is out of scope.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

# Stribeck speed fit v_s(h) = b1 exp(1000 b2 h + b3) + b4 (h in m)
STRIBECK_B = (4.8916, -7.91, 3.01, 3.40)
REFERENCE_SPEED = 13.89        # m/s, the speed mu is quoted at
SLIP_STATIC = 0.15
SLIP_DYNAMIC = 0.80
MU_FLOOR = 1e-3
H_NORM_MM = 1.0
AQUAPLANE_CENTER = 0.86
AQUAPLANE_WIDTH = 0.008

# frozen hydro-lift fit (data/hydro_coeffs.json of the reference)
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
    theta: float                  # macro-texture contact gain
    texture_amplitude_mm: float


SURFACE_ORDER = ("AC", "SMA", "OGFC")
SURFACES = {p.name: p for p in (SurfacePreset("AC", 1.00, 0.65), SurfacePreset("SMA", 1.09, 0.80),
                                SurfacePreset("OGFC", 1.21, 1.08))}
_THETA = np.array([SURFACES[n].theta for n in SURFACE_ORDER])


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


def _pow(x, p: float) -> np.ndarray:
    """x ** p elementwise with the C library's pow (numpy's scalar power),
    once per distinct base."""
    x = np.asarray(x, dtype=np.float64)
    u, inv = np.unique(x.reshape(-1), return_inverse=True)
    r = np.fromiter((math.pow(v, p) for v in u.tolist()), dtype=np.float64, count=len(u))
    return r[inv].reshape(x.shape)


@dataclass(frozen=True)
class HydroLiftModel:
    y_inf: float
    a: float
    p: float
    q: float
    c1: float
    c2: float

    def contact_ratio(self, v, h_mm):
        """Y_R: wet contact fraction with the aquaplaning gate."""
        u = np.asarray(v, dtype=np.float64) / REFERENCE_SPEED * np.asarray(h_mm, dtype=np.float64)
        base = self.y_inf + (1.0 - self.y_inf) * _pow(1.0 + _pow(u / self.a, self.p), -self.q)
        gate = 1.0 / (1.0 + np.exp(np.clip((u - AQUAPLANE_CENTER) / AQUAPLANE_WIDTH, -60.0, 60.0)))
        return base * gate

    def lift_ratio(self, v, h_mm):
        """Y_F: hydrodynamic lift fraction."""
        u = np.asarray(v, dtype=np.float64) / REFERENCE_SPEED * np.asarray(h_mm, dtype=np.float64)
        return np.minimum(self.c1 * _pow(np.maximum(u, 0.0), self.c2), 1.0)


@lru_cache(maxsize=1)
def default_hydro_model() -> HydroLiftModel:
    return HydroLiftModel(**HYDRO_COEFFS)


def stribeck_speed(h_w_m):
    """v_s(h) in m/s for a water film of h metres (scalar or array)."""
    h = np.asarray(h_w_m, dtype=np.float64)
    if (h < 0).any():
        raise ValueError("water film thickness must be non-negative")
    b1, b2, b3, b4 = STRIBECK_B
    out = b1 * np.exp(1000.0 * b2 * h + b3) + b4
    return float(out) if out.ndim == 0 else out


@lru_cache(maxsize=1)
def default_lugre_params(dry_static_mu=1.1048, dynamic_ratio=0.99, contact_length=0.15,
                         alpha=1.0, mu_c_ratio=0.75) -> LuGreParams:
    """(sigma0, mu_s) pinned by the two dry anchors (mu at 15 % and 80 % slip):
    linear in (1/mu_s, 1/sigma0), one 2x2 solve."""
    K = 7.0 / (6.0 * contact_length)
    v_s0 = stribeck_speed(0.0)
    rows, rhs = [], [1.0 / dry_static_mu, 1.0 / (dynamic_ratio * dry_static_mu)]
    for slip in (SLIP_STATIC, SLIP_DYNAMIC):
        q = mu_c_ratio + (1.0 - mu_c_ratio) * np.exp(-math.pow(slip * REFERENCE_SPEED / v_s0, alpha))
        rows.append([1.0 / q, K * (1.0 - slip) / slip])
    inv_mu_s, inv_sigma0 = np.linalg.solve(np.array(rows), np.array(rhs))
    mu_s = 1.0 / inv_mu_s
    return LuGreParams(1.0 / inv_sigma0, mu_s, mu_c_ratio * mu_s, alpha, contact_length)


def mu_table(surface_index, h_mm, v: float = REFERENCE_SPEED, slip: float = SLIP_STATIC,
             hydro: HydroLiftModel | None = None, params: LuGreParams | None = None) -> np.ndarray:
    """Effective friction coefficient for arrays of surfaces (indices into
    SURFACE_ORDER) and water films (mm) at speed v and slip ratio slip:
    mu = max(theta Y_R - Y_F, 0) * theta Y_R sigma0 z*, z* = v_r / lambda the
    bristle steady state, lambda = theta Y_R (sigma0 |v_r| / g(v_r) + K |w_r|)."""
    if v < 0:
        raise ValueError("speed must be non-negative")
    if not 0.0 <= slip <= 1.0:
        raise ValueError("slip ratio must lie in [0, 1]")
    hydro = hydro or default_hydro_model()
    prm = params or default_lugre_params()
    theta = _THETA[np.asarray(surface_index, dtype=np.int64)]
    h = np.asarray(h_mm, dtype=np.float64)
    v_r, w_r = slip * v, (1.0 - slip) * v
    if v_r == 0.0:
        return np.zeros(np.broadcast(theta, h).shape)
    y_r = hydro.contact_ratio(v, h)
    contact = np.maximum(theta * y_r - hydro.lift_ratio(v, h), 0.0)
    v_s = stribeck_speed(h * 1e-3)
    g = prm.mu_c_stribeck + (prm.mu_s_stribeck - prm.mu_c_stribeck) * np.exp(
        -_pow(np.abs(v_r / v_s), prm.alpha_stribeck))
    z_star = v_r / (theta * y_r * (prm.sigma0 * abs(v_r) / g + prm.K * abs(w_r)))
    mu = contact * theta * y_r * prm.sigma0 * z_star
    return np.where(contact == 0.0, 0.0, mu)


def mu_effective(surface_name: str, h_mm: float, v=REFERENCE_SPEED, slip=SLIP_STATIC,
                 hydro: HydroLiftModel | None = None, params: LuGreParams | None = None) -> float:
    """Scalar form of ``mu_table`` (the reference's signature)."""
    return float(mu_table(SURFACE_ORDER.index(surface(surface_name).name), h_mm, v, slip, hydro, params))


@dataclass(frozen=True)
class FrictionAssignment:
    surface: SurfacePreset
    water_film_mm: float
    mu_static: float
    mu_dynamic: float
    weather_token: np.ndarray  # [h/1mm, 1_AC, 1_SMA, 1_OGFC]


def weather_token(surface_name: str, h_mm: float) -> np.ndarray:
    tok = np.zeros(1 + len(SURFACE_ORDER))
    tok[0] = h_mm / H_NORM_MM
    tok[1 + SURFACE_ORDER.index(surface(surface_name).name)] = 1.0
    return tok


def assign_frictions(surfaces, films_mm, hydro=None, params=None) -> list[FrictionAssignment]:
    """Per-world assignments for parallel lists of surface names and films:
    mu_static / mu_dynamic at 15 % / 80 % slip, floored at MU_FLOOR."""
    idx = np.array([SURFACE_ORDER.index(surface(s).name) for s in surfaces], dtype=np.int64)
    h = np.asarray(films_mm, dtype=np.float64).reshape(-1)
    mu_s = np.maximum(mu_table(idx, h, REFERENCE_SPEED, SLIP_STATIC, hydro, params), MU_FLOOR)
    mu_d = np.maximum(mu_table(idx, h, REFERENCE_SPEED, SLIP_DYNAMIC, hydro, params), MU_FLOOR)
    tok = np.zeros((len(idx), 1 + len(SURFACE_ORDER)))
    tok[:, 0] = h / H_NORM_MM
    tok[np.arange(len(idx)), 1 + idx] = 1.0
    return [FrictionAssignment(SURFACES[SURFACE_ORDER[i]], float(hh), float(a), float(b), tok[w])
            for w, (i, hh, a, b) in enumerate(zip(idx, h, mu_s, mu_d))]


def assign_friction(surface_name: str, h_mm: float, hydro=None, params=None) -> FrictionAssignment:
    return assign_frictions([surface_name], [h_mm], hydro, params)[0]


def ground_material(f_surface: float, f_lon: float, f_lat: float):
    mu_s = min(1.0, f_surface * np.sqrt(f_lon * f_lat))
    return float(mu_s), float(0.95 * mu_s)


def effective_contact_mu(assignment: FrictionAssignment, ground_mu_s: float) -> float:
    return min(assignment.mu_static, ground_mu_s)
