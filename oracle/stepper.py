"""Float64 numpy restatement of the reference engine step (oracle, tests only).

Structure: one ``OracleEngine`` holding the (W, M) state dict in global
coordinates, with ``step`` / ``observe`` / ``teleport_reset``.  Each stage is a
free function over broadcastable arrays; the arithmetic of every expression is
kept in the reference's evaluation order (numpy never fuses a*b+c), which is
what makes the fixtures reproduce bit-for-bit on the same host.

Reference map (``/root/reference/pkg/src/drivegrid``):
  _check_actions / decode      engine.py:286-295, vehicle.py:162-173
  substep_dynamic              vehicle.py:176-191, 237-336
  substep_bicycle              vehicle.py:208-232
  ego_block                    observation.py:51-75
  road_block                   observation.py:78-125
  neighbour_block / ttc        observation.py:128-181, 235-293
  nearest_lane                 rewards.py:78-103
  dense_terms / edge_tau       rewards.py:106-176
  detectors / priority         rewards.py:181-268
  step tail / teleport_reset   engine.py:340-406, 472-509, 599-619
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from paper_2605_08528_b200 import params as P
from paper_2605_08528_b200.tables import build_tables, compact_subset, edge_mask_of, lane_mask_of

WORLD_CHUNK = 8


# --------------------------------------------------------------------------- physics

def decode(raw):
    out = np.empty_like(raw)
    out[..., 0] = np.clip(raw[..., 0], 0.0, 1.0)
    out[..., 1] = np.clip(raw[..., 1], -1.0, 1.0)
    out[..., 2] = np.clip(raw[..., 2], 0.0, 1.0)
    return out


def _brake(wheel, cmd, latch, tau):
    sgn = np.where(np.abs(wheel) >= P.WHEEL_SPEED_LATCH_EPS, np.sign(wheel), latch)
    return -sgn * cmd * tau, sgn


def substep_dynamic(s: dict, act, mu, vp: P.VehicleParams, dt: float) -> dict:
    thr, steer, brk = act[..., 0], act[..., 1], act[..., 2]
    tau_s = np.clip(vp.kp_steer * (vp.theta_max * steer - s["steer_angle"]) - vp.kd_steer * s["steer_rate"],
                    -vp.tau_steer_max, vp.tau_steer_max)
    rate = s["steer_rate"] + (tau_s / vp.steer_inertia) * dt
    ang = s["steer_angle"] + rate * dt
    lim = 1.05 * vp.theta_max
    ang_c = np.clip(ang, -lim, lim)
    rate = np.where(ang_c == ang, rate, 0.0)
    ang = ang_c

    vx, vy, om = s["v_x"], s["v_y"], s["yaw_rate"]
    a_f = 0.5 * vp.wheelbase - vp.com_offset
    b_r = 0.5 * vp.wheelbase + vp.com_offset
    tbf, latch_f = _brake(s["wheel_front"], brk, s["brake_sign_front"], vp.tau_brake_front)
    tbr, latch_r = _brake(s["wheel_rear"], brk, s["brake_sign_rear"], vp.tau_brake_rear)
    t_front = 2.0 * (vp.tau_drive_max * thr + tbf)
    t_rear = 2.0 * tbr
    fxf0 = t_front / vp.wheel_radius
    fxr0 = t_rear / vp.wheel_radius
    den = np.maximum(vx, P.SLIP_SPEED_FLOOR)
    fyf0 = vp.cornering_stiffness * (ang - (vy + a_f * om) / den)
    fyr0 = vp.cornering_stiffness * (-(vy - b_r * om) / den)

    cap = mu * (0.5 * vp.chassis_mass * P.GRAVITY)
    nf = np.sqrt(fxf0 ** 2 + fyf0 ** 2)
    nr = np.sqrt(fxr0 ** 2 + fyr0 ** 2)
    kf = np.where(nf > cap, cap / np.maximum(nf, 1e-12), 1.0)
    kr = np.where(nr > cap, cap / np.maximum(nr, 1e-12), 1.0)
    fxf, fyf = fxf0 * kf, fyf0 * kf
    fxr, fyr = fxr0 * kr, fyr0 * kr

    cd, sd = np.cos(ang), np.sin(ang)
    m = vp.chassis_mass
    ax = (fxf * cd - fyf * sd + fxr) / m + vy * om
    ay = (fyf * cd + fxf * sd + fyr - vp.lambda_lat * vy) / m - vx * om
    omd = (a_f * (fyf * cd + fxf * sd) - b_r * fyr - vp.lambda_yaw * om) / vp.yaw_inertia
    vx1 = vx + ax * dt
    vy1 = vy + ay * dt
    om1 = om + omd * dt
    vx1 = np.where((brk > 0.0) & (vx >= 0.0) & (vx1 < 0.0), 0.0, vx1)

    yaw = s["yaw"]
    cy, sy = np.cos(yaw), np.sin(yaw)
    out = dict(s)
    out["x"] = s["x"] + (vx1 * cy - vy1 * sy) * dt
    out["y"] = s["y"] + (vx1 * sy + vy1 * cy) * dt
    out["yaw"] = yaw + om1 * dt

    i_axle = 2.0 * vp.wheel_inertia
    roll_f = ((vy1 + a_f * om1) * sd + vx1 * cd) / vp.wheel_radius
    roll_r = vx1 / vp.wheel_radius
    spin_f = s["wheel_front"] + (t_front - fxf * vp.wheel_radius) / i_axle * dt
    spin_r = s["wheel_rear"] + (t_rear - fxr * vp.wheel_radius) / i_axle * dt
    spin_f = np.where((brk > 0.0) & (spin_f * latch_f < 0.0), 0.0, spin_f)
    spin_r = np.where((brk > 0.0) & (spin_r * latch_r < 0.0), 0.0, spin_r)
    out["wheel_front"] = np.clip(np.where(nf > cap, spin_f, roll_f), -P.WHEEL_SPEED_LIMIT, P.WHEEL_SPEED_LIMIT)
    out["wheel_rear"] = np.clip(np.where(nr > cap, spin_r, roll_r), -P.WHEEL_SPEED_LIMIT, P.WHEEL_SPEED_LIMIT)
    out["v_x"], out["v_y"], out["yaw_rate"] = vx1, vy1, om1
    out["steer_angle"], out["steer_rate"] = ang, rate
    out["brake_sign_front"], out["brake_sign_rear"] = latch_f, latch_r
    return out


def substep_bicycle(s: dict, act, vp: P.VehicleParams, bp: P.BicycleParams, dt: float) -> dict:
    thr, steer, brk = act[..., 0], act[..., 1], act[..., 2]
    delta = steer * P.BICYCLE_STEER_MAX
    v = s["v_x"]
    v1 = np.maximum(v + (thr * bp.a_max - brk * bp.b_max - np.sign(v) * bp.c_roll) * dt, 0.0)
    yaw = s["yaw"]
    rate = v1 * np.tan(delta) / vp.wheelbase
    out = dict(s)
    out["x"] = s["x"] + v1 * np.cos(yaw) * dt
    out["y"] = s["y"] + v1 * np.sin(yaw) * dt
    out["yaw"] = yaw + rate * dt
    out["v_x"] = v1
    out["v_y"] = np.zeros_like(v1)
    out["yaw_rate"] = rate
    out["steer_angle"] = delta
    out["steer_rate"] = np.zeros_like(v1)
    out["wheel_front"] = v1 / vp.wheel_radius
    out["wheel_rear"] = v1 / vp.wheel_radius
    return out


# --------------------------------------------------------------------------- observation

def rot(dx, dy, c, s):
    """World offset -> body frame given cos/sin of yaw."""
    return c * dx + s * dy, -s * dx + c * dy


def ego_block(px, py, c, s, vx, vy, gx, gy, weather, oc: P.ObsConfig):
    dxb, dyb = rot(gx - px, gy - py, c, s)
    hdg = np.arctan2(dyb, dxb)
    cols = [dxb / oc.bbox_half, dyb / oc.bbox_half, np.sin(hdg), np.cos(hdg),
            np.sqrt(dxb * dxb + dyb * dyb) / oc.bbox_half, vx / oc.speed_norm, vy / oc.speed_norm]
    if oc.include_weather:
        cols += [np.broadcast_to(weather[..., k], dxb.shape) for k in range(4)]
    return np.stack(cols, axis=-1)


def road_block(px, py, c, s, mid, dirs, codes, mask, oc: P.ObsConfig):
    """Ordered compaction of the segments within the road radius; rows carry
    [dxb/r, dyb/r, type/20, dir_b]; the compaction order is the segment index."""
    dx = mid[..., 0] - px[..., None]
    dy = mid[..., 1] - py[..., None]
    cand = (dx * dx + dy * dy <= oc.road_radius ** 2) & mask
    nP = mid.shape[-2]
    take = min(oc.k_road, nP)
    rank = np.cumsum(cand, axis=-1) - 1
    hit = cand & (rank < take)
    out = np.zeros(px.shape + (oc.k_road, 5))
    w_i, m_i, p_i = np.nonzero(np.broadcast_to(hit, dx.shape))
    slot = rank[w_i, m_i, p_i]
    cs, ss = c[w_i, m_i], s[w_i, m_i]
    ddx, ddy = dx[w_i, m_i, p_i], dy[w_i, m_i, p_i]
    dirx, diry = dirs[w_i, 0, p_i, 0], dirs[w_i, 0, p_i, 1]
    xb, yb = rot(ddx, ddy, cs, ss)
    bx, by = rot(dirx, diry, cs, ss)
    out[w_i, m_i, slot, 0] = xb / oc.road_radius
    out[w_i, m_i, slot, 1] = yb / oc.road_radius
    out[w_i, m_i, slot, 2] = codes[w_i, 0, p_i].astype(np.float64) / oc.type_norm
    out[w_i, m_i, slot, 3] = bx
    out[w_i, m_i, slot, 4] = by
    return out


def hull(px, py, c, s, d):
    """Three circle centres along the heading, (..., 3) each."""
    off = np.array([-1.0, 0.0, 1.0]) * np.asarray(d)[..., None]
    return px[..., None] + off * c[..., None], py[..., None] + off * s[..., None]


def pair_ttc(dx, dy, ux, uy, ce, se, cn, sn, de, dn, rsum, tmax):
    """Swept 3x3 circle closest approach (observation.py:128-181); inputs
    broadcast over (..., ego, other)."""
    off = np.array([-1.0, 0.0, 1.0])
    oe = off[:, None] * np.asarray(de)[..., None, None]
    on = off[None, :] * np.asarray(dn)[..., None, None]
    qx = dx[..., None, None] + on * cn[..., None, None] - oe * ce[..., None, None]
    qy = dy[..., None, None] + on * sn[..., None, None] - oe * se[..., None, None]
    a = (ux * ux + uy * uy)[..., None, None]
    b = 2.0 * (qx * ux[..., None, None] + qy * uy[..., None, None])
    rr = rsum[..., None, None]
    cc = qx * qx + qy * qy - rr * rr
    disc = b * b - 4.0 * a * cc
    moving = a >= 1e-12
    root = np.sqrt(np.maximum(disc, 0.0))
    a2 = 2.0 * np.where(moving, a, 1.0)
    t_in = (-b - root) / a2
    t_out = (-b + root) / a2
    t = np.where(moving & (disc >= 0.0) & (t_out >= 0.0), np.maximum(t_in, 0.0), tmax)
    t = np.where(~moving & (cc < 0.0), 0.0, t)
    t = np.min(np.clip(t, 0.0, tmax), axis=(-2, -1))
    return np.where(ce * dx + se * dy < 0.0, tmax, t)


def neighbour_block(px, py, yaw, c, s, vx, vy, vwx, vwy, length, width, r, d, alive,
                    oc: P.ObsConfig):
    W, M = px.shape
    dx = px[:, None, :] - px[:, :, None]
    dy = py[:, None, :] - py[:, :, None]
    dist = np.sqrt(dx * dx + dy * dy)
    dist = np.where(alive[:, None, :] & ~np.eye(M, dtype=bool)[None], dist, np.inf)
    take = min(oc.k_vehicles, M)
    sel = np.argsort(dist, axis=-1, kind="stable")[..., :take]
    ok = np.isfinite(np.take_along_axis(dist, sel, axis=-1))

    def pick(a):
        return np.take_along_axis(np.broadcast_to(a[:, None, :], (W, M, M)), sel, axis=-1)

    sdx, sdy = np.take_along_axis(dx, sel, axis=-1), np.take_along_axis(dy, sel, axis=-1)
    xb, yb = rot(sdx, sdy, c[..., None], s[..., None])
    turn = pick(yaw) - yaw[..., None]
    wrap = np.arctan2(np.sin(turn), np.cos(turn))
    nvx, nvy = pick(vx), pick(vy)
    n_len, n_wid = pick(length), pick(width)
    ttc = pair_ttc(sdx, sdy, pick(vwx) - vwx[..., None], pick(vwy) - vwy[..., None],
                   c[..., None], s[..., None], pick(c), pick(s), d[..., None], pick(d),
                   r[..., None] + pick(r), oc.ttc_max)
    feats = np.stack([xb / oc.bbox_half, yb / oc.bbox_half, n_len / oc.bbox_half,
                      n_wid / oc.bbox_half, wrap / np.pi, np.sqrt(nvx * nvx + nvy * nvy) / oc.speed_norm,
                      ttc / oc.ttc_max], axis=-1)
    feats = np.where(ok[..., None], feats, 0.0)
    tmin = np.min(np.where(ok, ttc, oc.ttc_max), axis=-1) if take else np.full((W, M), oc.ttc_max)
    rows = np.zeros((W, M, oc.k_vehicles, 7))
    rows[:, :, :take] = feats
    return rows, tmin


# --------------------------------------------------------------------------- rewards / events

def nearest_lane(px, py, mid, dirs, mask, hl):
    ex = px[..., None] - mid[..., 0]
    ey = py[..., None] - mid[..., 1]
    along = ex * dirs[..., 0] + ey * dirs[..., 1]
    lat = dirs[..., 0] * ey - dirs[..., 1] * ex
    over = np.maximum(np.abs(along) - hl, 0.0)
    d2 = np.where(mask, over * over + lat * lat, np.inf)
    k = np.argmin(d2, axis=-1)[..., None]
    dist = np.sqrt(np.take_along_axis(d2, k, axis=-1)[..., 0])
    lat_k = np.take_along_axis(lat, k, axis=-1)[..., 0]
    tx = np.take_along_axis(np.broadcast_to(dirs[..., 0], d2.shape), k, axis=-1)[..., 0]
    ty = np.take_along_axis(np.broadcast_to(dirs[..., 1], d2.shape), k, axis=-1)[..., 0]
    none = ~np.isfinite(dist)
    return dist, np.where(none, 0.0, lat_k), np.where(none, 0.0, tx), np.where(none, 0.0, ty)


def edge_tau(px, py, c, s, vx, mid, mask, rc: P.RewardConfig):
    xb = c[..., None] * (mid[..., 0] - px[..., None]) + s[..., None] * (mid[..., 1] - py[..., None])
    gap = np.min(np.where(mask & (xb > 0.0) & (xb <= rc.edge_range), xb, np.inf), axis=-1)
    return gap / np.maximum(vx, 0.1)


def dense_terms(ppx, ppy, px, py, yaw, c, s, vx, vy, gx, gy, tmin, lane, edge, rc: P.RewardConfig):
    dist, lat, tx, ty = nearest_lane(px, py, lane["mid"], lane["dir"], lane["mask"], lane["half_len"])
    sgn = np.where(tx * (gx - px) + ty * (gy - py) >= 0.0, 1.0, -1.0)
    tx, ty = tx * sgn, ty * sgn
    prog = np.clip((px - ppx) * tx + (py - ppy) * ty, -rc.progress_clamp, rc.progress_clamp) * rc.progress_weight
    align = np.maximum(0.0, np.cos(yaw - np.arctan2(ty, tx)))
    quality = np.exp(-((lat / rc.lane_sigma) ** 2)) * (
        (1.0 - rc.lane_heading_weight) + rc.lane_heading_weight * align)
    has = np.isfinite(dist)
    lane_t = np.where(has, rc.lane_weight * quality, 0.0)
    prog = np.where(has, prog, 0.0)
    off = np.where(has & ((np.abs(lat) > rc.offroad_lat_limit) | (dist > rc.offroad_dist_limit)),
                   -rc.offroad_weight, 0.0)
    idle = np.where(np.sqrt(vx ** 2 + vy ** 2) < rc.idle_speed, -rc.idle_weight, 0.0)
    ttc_v = -np.minimum(rc.ttc_vehicle_alpha / np.maximum(tmin, rc.ttc_floor), rc.ttc_vehicle_pmax)
    tau = edge_tau(px, py, c, s, vx, edge["mid"], edge["mask"], rc)
    ttc_e = np.where(np.isfinite(tau), -np.minimum(rc.ttc_edge_alpha / np.maximum(tau, rc.ttc_floor),
                                                   rc.ttc_edge_pmax), 0.0)
    terms = {"progress": prog, "lane": lane_t, "offroad": off, "idle": idle,
             "ttc_vehicle": ttc_v, "ttc_edge": ttc_e}
    terms["total"] = prog + lane_t + off + idle + ttc_v + ttc_e
    return terms


def edge_overlap(px, py, c, s, r, d, edge):
    """Any hull circle closer than r to a road-edge box (rewards.py:208-223)."""
    hx, hy = hull(px, py, c, s, d)
    mid, dirs = edge["mid"], edge["dir"]
    qx = hx[..., None] - mid[..., None, :, 0]
    qy = hy[..., None] - mid[..., None, :, 1]
    ax, ay = dirs[..., None, :, 0], dirs[..., None, :, 1]
    along = qx * ax + qy * ay
    lat = ax * qy - ay * qx
    hl, hw = edge["half_len"][..., None, :], edge["half_wid"][..., None, :]
    du = along - np.clip(along, -hl, hl)
    dv = lat - np.clip(lat, -hw, hw)
    hit = (du * du + dv * dv < np.asarray(r)[..., None, None] ** 2) & edge["mask"][..., None, :]
    return hit.any(axis=(-2, -1))


def hull_contact(px, py, c, s, r, d, alive, age, warmup):
    """Per-agent overlap with any other alive hull, after the warmup (rewards.py:226-250)."""
    hx, hy = hull(px, py, c, s, d)                       # (W, M, 3)
    ex = hx[:, :, None, :, None] - hx[:, None, :, None, :]  # (W, M, M, 3, 3)
    ey = hy[:, :, None, :, None] - hy[:, None, :, None, :]
    rs = (r[:, :, None] + r[:, None, :])[..., None, None]
    touch = (ex * ex + ey * ey < rs * rs).any(axis=(-2, -1))
    M = px.shape[1]
    pair = alive[:, :, None] & alive[:, None, :] & ~np.eye(M, dtype=bool)[None]
    return (touch & pair).any(axis=-1) & (age >= warmup)


def priority(goal, crash, edge_hit, contact):
    rsn = np.where(contact, P.REASON_COLLISION, P.REASON_NONE)
    rsn = np.where(edge_hit, P.REASON_LANE_FORBIDDEN, rsn)
    rsn = np.where(crash, P.REASON_CRASH, rsn)
    return np.where(goal, P.REASON_GOAL, rsn)


def one_shot(rsn, rc: P.RewardConfig):
    out = np.zeros(np.shape(rsn))
    out = np.where(rsn == P.REASON_GOAL, rc.goal_weight, out)
    out = np.where(rsn == P.REASON_COLLISION, -rc.collision_weight, out)
    out = np.where(rsn == P.REASON_CRASH, -rc.crash_weight, out)
    return np.where(rsn == P.REASON_LANE_FORBIDDEN, -rc.lane_forbidden_weight, out)


# --------------------------------------------------------------------------- integer decisions

def road_order(px, py, mid, mask, oc: P.ObsConfig):
    """Road slot -> segment index: the stable argsort of ~cand, first
    min(K_r, P) entries (observation.py:92-99); n = candidates kept."""
    dx = mid[..., 0] - px[..., None]
    dy = mid[..., 1] - py[..., None]
    cand = (dx * dx + dy * dy <= oc.road_radius ** 2) & mask
    take = min(oc.k_road, mid.shape[-2])
    order = np.argsort(~cand, axis=-1, kind="stable")[..., :take]
    return order, np.minimum(cand.sum(axis=-1), take)


def neighbour_order(px, py, alive, oc: P.ObsConfig):
    """Neighbour rank -> agent index: stable argsort of the distances with
    dead agents and self at inf, first min(K_v, M) (observation.py:239-249);
    n = finite entries."""
    M = px.shape[1]
    dx = px[:, None, :] - px[:, :, None]
    dy = py[:, None, :] - py[:, :, None]
    dist = np.sqrt(dx * dx + dy * dy)
    dist = np.where(alive[:, None, :], dist, np.inf)
    dist = np.where(np.eye(M, dtype=bool)[None], np.inf, dist)
    take = min(oc.k_vehicles, M)
    sel = np.argsort(dist, axis=-1, kind="stable")[..., :take]
    return sel, np.isfinite(np.take_along_axis(dist, sel, axis=-1)).sum(axis=-1)


def lane_index(px, py, lane):
    """np.argmin (first index on ties) of the point-to-segment d2 over the
    compacted lane subset (rewards.py:87-94); -1 where no lane exists."""
    ex = px[..., None] - lane["mid"][..., 0]
    ey = py[..., None] - lane["mid"][..., 1]
    along = ex * lane["dir"][..., 0] + ey * lane["dir"][..., 1]
    lat = lane["dir"][..., 0] * ey - lane["dir"][..., 1] * ex
    over = np.maximum(np.abs(along) - lane["half_len"], 0.0)
    d2 = np.where(lane["mask"], over * over + lat * lat, np.inf)
    k = np.argmin(d2, axis=-1) if d2.shape[-1] else np.zeros(px.shape, dtype=np.int64)
    best = np.take_along_axis(d2, k[..., None], axis=-1)[..., 0] if d2.shape[-1] else np.full(px.shape, np.inf)
    return np.where(np.isfinite(best), k, -1)


@dataclass
class IndexRecord:
    """The integer decisions of one step, in the kernel's index_out terms."""
    lane: np.ndarray        # (W, M) nearest-lane index, -1: none / not alive before the step
    road: np.ndarray        # (W, M, take_road) slot -> segment
    road_n: np.ndarray      # (W, M)
    veh: np.ndarray         # (W, M, take_veh) rank -> agent
    veh_n: np.ndarray       # (W, M)


# --------------------------------------------------------------------------- engine

@dataclass
class OracleStep:
    obs: np.ndarray
    rewards: np.ndarray
    dones: np.ndarray
    events: dict
    info: dict


class OracleEngine:
    """CPU twin of the GPU engine over the same host tables."""

    def __init__(self, worlds, scenes, assignment, frictions, config: P.SimConfig,
                 obs_config=None, reward_config=None, params=None, bicycle=None, num_workers=None):
        self.config = config
        self.obs_config = obs_config or P.ObsConfig()
        self.reward_config = reward_config or P.RewardConfig()
        self.params = params or P.VehicleParams()
        self.bicycle = bicycle or P.BicycleParams()
        t = build_tables(worlds, scenes, assignment, frictions, config, self.params)
        self.tables = t
        self.worlds = worlds
        self.W, self.M = t.W, t.M
        gm = worlds.midpoints + worlds.grid_offsets[:, None, :]
        self.seg = {"mid": gm[:, None], "dir": worlds.directions[:, None],
                    "type": worlds.type_codes[:, None], "mask": worlds.mask[:, None]}
        self.lane = compact_subset(worlds, lane_mask_of(worlds.type_codes, worlds.mask))
        self.edge = compact_subset(worlds, edge_mask_of(worlds.type_codes, worlds.mask))
        self.mu_eff, self.weather = t.mu_eff, t.weather
        self.valid, self.alive = t.valid.copy(), t.valid.copy()
        self.start_xy, self.goal_xy, self.start_yaw = t.start_xy.copy(), t.goal_xy.copy(), t.start_yaw.copy()
        self.length, self.width, self.r_hull, self.d_hull = t.length, t.width, t.r_hull, t.d_hull
        self.state = {k: v.copy() for k, v in t.state0.items()}
        self.reason = np.zeros((self.W, self.M), dtype=np.int8)
        self.spawn_step = np.zeros((self.W, self.M), dtype=np.int64)
        self.event_seen = {k: np.zeros((self.W, self.M), dtype=bool) for k in P.EVENT_TYPES}
        self.step_count = 0
        self.record_indices = False   # step() adds info["indices"] (IndexRecord)
        workers = config.effective_workers if num_workers is None else max(1, num_workers)
        self._pool = ThreadPoolExecutor(workers) if workers > 1 else None

    # ----------------------------------------------------------------- helpers
    def _chunks(self):
        return [slice(a, min(a + WORLD_CHUNK, self.W)) for a in range(0, self.W, WORLD_CHUNK)]

    def _map(self, fn):
        chunks = self._chunks()
        if self._pool is None or len(chunks) == 1:
            for ch in chunks:
                fn(ch)
        else:
            list(self._pool.map(fn, chunks))

    def _kin(self):
        st = self.state
        c, s = np.cos(st["yaw"]), np.sin(st["yaw"])
        vwx = st["v_x"] * c - st["v_y"] * s
        vwy = st["v_x"] * s + st["v_y"] * c
        return c, s, vwx, vwy

    # ----------------------------------------------------------------- observe
    def _observe(self):
        oc = self.obs_config
        st = self.state
        c, s, vwx, vwy = self._kin()
        obs = np.empty((self.W, self.M, oc.obs_dim), dtype=np.float32)
        tmin = np.empty((self.W, self.M))
        e0, e1 = oc.ego_dim, oc.ego_dim + 5 * oc.k_road

        def work(ch):
            px, py, yaw = st["x"][ch], st["y"][ch], st["yaw"][ch]
            obs[ch, :, :e0] = ego_block(px, py, c[ch], s[ch], st["v_x"][ch], st["v_y"][ch],
                                        self.goal_xy[ch][..., 0], self.goal_xy[ch][..., 1],
                                        self.weather[ch][:, None, :], oc)
            road = road_block(px, py, c[ch], s[ch], self.seg["mid"][ch], self.seg["dir"][ch],
                              self.seg["type"][ch], self.seg["mask"][ch], oc)
            obs[ch, :, e0:e1] = road.reshape(road.shape[:2] + (-1,))
            veh, tm = neighbour_block(px, py, yaw, c[ch], s[ch], st["v_x"][ch], st["v_y"][ch],
                                      vwx[ch], vwy[ch], self.length[ch], self.width[ch],
                                      self.r_hull[ch], self.d_hull[ch], self.alive[ch], oc)
            obs[ch, :, e1:] = veh.reshape(veh.shape[:2] + (-1,))
            tmin[ch] = tm

        self._map(work)
        return obs, tmin

    def observe(self):
        return self._observe()[0]

    # ----------------------------------------------------------------- step
    def check_actions(self, actions):
        a = np.asarray(actions, dtype=np.float64)
        want = (self.W, self.M, 3)
        if a.shape != want:
            raise ValueError(f"actions shape {a.shape}, expected {want}")
        bad = ~np.isfinite(a)
        if bad.any():
            w, m, _ = np.argwhere(bad)[0]
            raise ValueError(f"non-finite action for world {w} agent {m}")
        return a

    def step(self, actions) -> OracleStep:
        cfg, rc = self.config, self.reward_config
        act = decode(self.check_actions(actions))
        st = self.state
        ppx, ppy = st["x"], st["y"]

        if cfg.dynamics_mode == "bicycle":
            new = substep_bicycle(st, act, self.params, self.bicycle, cfg.control_dt)
        else:
            new = st
            mu = self.mu_eff[:, None]
            for _ in range(cfg.decimation):
                new = substep_dynamic(new, act, mu, self.params, cfg.physics_dt)
        self.state = st = {k: np.where(self.alive, new[k], st[k]) for k in P.STATE_FIELDS}

        obs, tmin = self._observe()
        alive_pre = self.alive.copy()
        snapshot = {k: v.copy() for k, v in st.items()}
        indices = self.index_record(st, alive_pre) if self.record_indices else None

        # rewards and events against the pre-step alive mask
        W, M = self.W, self.M
        c, s, _, _ = self._kin()
        age = self.step_count - self.spawn_step
        names = (*P.DENSE_TERMS, "total")
        terms = {k: np.empty((W, M)) for k in names}
        ev = {k: np.empty((W, M), dtype=bool) for k in P.EVENT_TYPES}

        def work(ch):
            px, py = st["x"][ch], st["y"][ch]
            vx, vy = st["v_x"][ch], st["v_y"][ch]
            gx, gy = self.goal_xy[ch][..., 0], self.goal_xy[ch][..., 1]
            lane = {k: v[ch] for k, v in self.lane.items()}
            edge = {k: v[ch] for k, v in self.edge.items()}
            t = dense_terms(ppx[ch], ppy[ch], px, py, st["yaw"][ch], c[ch], s[ch], vx, vy, gx, gy,
                            tmin[ch], lane, edge, rc)
            for k in names:
                terms[k][ch] = t[k]
            ddx, ddy = gx - px, gy - py
            ev["goal"][ch] = np.sqrt(ddx * ddx + ddy * ddy) <= rc.goal_radius
            sx, sy = px - self.start_xy[ch][..., 0], py - self.start_xy[ch][..., 1]
            finite = np.isfinite(px) & np.isfinite(py) & np.isfinite(vx) & np.isfinite(vy)
            ev["crash"][ch] = ((np.sqrt(sx * sx + sy * sy) > rc.crash_drift_limit) | ~finite
                               | (np.sqrt(vx ** 2 + vy ** 2) > P.CRASH_SPEED_LIMIT))
            ev["lane_forbidden"][ch] = edge_overlap(px, py, c[ch], s[ch], self.r_hull[ch],
                                                    self.d_hull[ch], edge)
            ev["collision"][ch] = hull_contact(px, py, c[ch], s[ch], self.r_hull[ch], self.d_hull[ch],
                                               self.alive[ch], age[ch], rc.collision_warmup_steps)

        self._map(work)
        for k in P.EVENT_TYPES:
            ev[k] &= self.alive & ~self.event_seen[k]
        rsn = priority(ev["goal"], ev["crash"], ev["lane_forbidden"], ev["collision"])
        events = {"goal": rsn == P.REASON_GOAL, "collision": rsn == P.REASON_COLLISION,
                  "crash": rsn == P.REASON_CRASH, "lane_forbidden": rsn == P.REASON_LANE_FORBIDDEN}
        for k in P.EVENT_TYPES:
            self.event_seen[k] |= events[k]
        rewards = np.where(self.alive, terms["total"] + one_shot(rsn, rc), 0.0)
        terms = {k: np.where(self.alive, v, 0.0) for k, v in terms.items()}
        if cfg.invincible:
            dones = np.zeros((W, M), dtype=bool)
        else:
            dones = rsn != P.REASON_NONE
            self.reason = np.where(dones & (self.reason == P.REASON_NONE), rsn, self.reason).astype(np.int8)

        # tail: timeout, park, alive
        self.step_count += 1
        timeout = self.alive.copy() if self.step_count >= cfg.episode_len else np.zeros((W, M), dtype=bool)
        finished = dones | timeout
        self.reason = np.where(timeout & (self.reason == P.REASON_NONE), P.REASON_TIMEOUT,
                               self.reason).astype(np.int8)
        park = dones & ~timeout
        if park.any():
            for k in P.STATE_FIELDS:
                st[k] = np.where(park, 1.0 if k.startswith("brake_sign") else 0.0, st[k])
            st["x"] = np.where(park, self.tables.grid_offsets[:, 0][:, None] + P.OFFSTAGE_X, st["x"])
            st["y"] = np.where(park, self.tables.grid_offsets[:, 1][:, None], st["y"])
        self.alive &= ~finished
        info = {"alive": self.alive.copy(), "alive_pre": alive_pre, "state": snapshot,
                "reason": self.reason.copy(), "reward_terms": terms, "ttc_min": tmin,
                "step": self.step_count}
        if indices is not None:
            info["indices"] = indices
        return OracleStep(obs, rewards, finished, events, info)

    def index_record(self, st, alive) -> IndexRecord:
        """Integer decisions on the post-physics state ``st`` with the alive
        mask the step used (world chunks like the float work)."""
        oc = self.obs_config
        W, M = self.W, self.M
        take_r = min(oc.k_road, self.seg["mid"].shape[-2])
        take_v = min(oc.k_vehicles, M)
        rec = IndexRecord(np.full((W, M), -1, np.int64), np.zeros((W, M, take_r), np.int64),
                          np.zeros((W, M), np.int64), np.zeros((W, M, take_v), np.int64),
                          np.zeros((W, M), np.int64))

        def work(ch):
            px, py = st["x"][ch], st["y"][ch]
            rec.road[ch], rec.road_n[ch] = road_order(px, py, self.seg["mid"][ch], self.seg["mask"][ch], oc)
            rec.veh[ch], rec.veh_n[ch] = neighbour_order(px, py, alive[ch], oc)
            lk = lane_index(px, py, {k: v[ch] for k, v in self.lane.items()})
            rec.lane[ch] = np.where(alive[ch], lk, -1)

        self._map(work)
        return rec

    # ----------------------------------------------------------------- reset
    def teleport_reset(self, mask, new_starts=None, new_goals=None, new_headings=None):
        mask = np.asarray(mask, dtype=bool) & self.valid
        if new_starts is not None:
            self.start_xy = np.where(mask[..., None], new_starts, self.start_xy)
        if new_goals is not None:
            self.goal_xy = np.where(mask[..., None], new_goals, self.goal_xy)
        if new_headings is not None:
            self.start_yaw = np.where(mask, new_headings, self.start_yaw)
        st = self.state
        for k in P.STATE_FIELDS:
            st[k] = np.where(mask, 1.0 if k.startswith("brake_sign") else 0.0, st[k])
        st["x"] = np.where(mask, self.start_xy[..., 0], st["x"])
        st["y"] = np.where(mask, self.start_xy[..., 1], st["y"])
        st["yaw"] = np.where(mask, self.start_yaw, st["yaw"])
        self.alive |= mask
        self.reason = np.where(mask, P.REASON_NONE, self.reason).astype(np.int8)
        self.spawn_step = np.where(mask, self.step_count, self.spawn_step)
        for k in P.EVENT_TYPES:
            self.event_seen[k] &= ~mask

    def env_reset(self):
        """``EnvHandle.reset`` semantics (env.py:37-46), including the
        spawn_step-before-zero quirk."""
        self.teleport_reset(self.valid)
        self.step_count = 0
        return self.observe()
