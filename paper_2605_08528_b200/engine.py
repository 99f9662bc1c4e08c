"""GPU batch engine: the drop-in for ``drivegrid.engine.Engine``.

Construction mirrors the reference signature (engine.py:151-162) and builds
the same host tables; per step, ``step()`` issues ONE fused kernel through the
C ABI (``dg_step``) that runs decode -> 4 physics substeps -> observation ->
rewards/events -> timeout/park tail for every world.

Array namespace follows the caller:
  * numpy actions  -> numpy outputs (host copies; the reference's exact
    semantics, including raising on non-finite actions before mutating);
  * torch CUDA actions -> torch CUDA outputs that stay in HBM (the fast path;
    non-finite actions are flagged on the device, see ``check_actions``).

State lives on the device in float64 global coordinates, laid out
``[12][W][M]`` (``state_tensor``); ``engine.state`` returns host copies keyed
like the reference.  There is no CPU fallback: constructing an Engine without
a CUDA device or without the native library raises.
"""

from __future__ import annotations

import ctypes as ct
import os
import time
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .params import (CRASH_SPEED_LIMIT, DENSE_TERMS, EVENT_TYPES, GRAVITY, OFFSTAGE_X, PHASES,
                     STATE_FIELDS, BicycleParams, ObsConfig, RewardConfig, SimConfig, VehicleParams)
from .spatial import build_scene_index
from .tables import build_tables, compact_subset, edge_mask_of, lane_mask_of
from .worldgen import DeviceWorldBatch
from .worldgen import engine_tables as device_engine_tables

TERM_NAMES = (*DENSE_TERMS, "total")


def _ptr(t: torch.Tensor | None):
    return None if t is None else ct.c_void_p(t.data_ptr())


def _align16(n: int) -> int:
    return (n + 15) & ~15


def make_consts(cfg: SimConfig, oc: ObsConfig, rc: RewardConfig, vp: VehicleParams,
                bp: BicycleParams) -> N.DgConsts:
    """Scalar constants with the reference's Python-side expression order."""
    k = N.DgConsts()
    vals = dict(
        physics_dt=cfg.physics_dt, control_dt=cfg.control_dt,
        kp_steer=vp.kp_steer, kd_steer=vp.kd_steer, theta_max=vp.theta_max,
        tau_steer_max=vp.tau_steer_max, steer_inertia=vp.steer_inertia,
        steer_limit=1.05 * vp.theta_max,
        a_f=0.5 * vp.wheelbase - vp.com_offset, b_r=0.5 * vp.wheelbase + vp.com_offset,
        tau_drive_max=vp.tau_drive_max, tau_brake_front=vp.tau_brake_front,
        tau_brake_rear=vp.tau_brake_rear, wheel_radius=vp.wheel_radius,
        cornering_stiffness=vp.cornering_stiffness, f_z=0.5 * vp.chassis_mass * GRAVITY,
        chassis_mass=vp.chassis_mass, lambda_lat=vp.lambda_lat, lambda_yaw=vp.lambda_yaw,
        yaw_inertia=vp.yaw_inertia, i_axle=2.0 * vp.wheel_inertia, wheelbase=vp.wheelbase,
        bic_a_max=bp.a_max, bic_b_max=bp.b_max, bic_c_roll=bp.c_roll,
        bic_steer_max=float(np.deg2rad(30.0)),
        road_radius=oc.road_radius, road_radius_sq=oc.road_radius ** 2, bbox_half=oc.bbox_half,
        speed_norm=oc.speed_norm, type_norm=oc.type_norm, ttc_max=oc.ttc_max,
        goal_radius=rc.goal_radius, goal_weight=rc.goal_weight,
        collision_weight=rc.collision_weight, crash_weight=rc.crash_weight,
        crash_drift_limit=rc.crash_drift_limit, lane_forbidden_weight=rc.lane_forbidden_weight,
        progress_weight=rc.progress_weight, progress_clamp=rc.progress_clamp,
        lane_weight=rc.lane_weight, lane_sigma=rc.lane_sigma,
        lane_heading_weight=rc.lane_heading_weight,
        lane_heading_base=1.0 - rc.lane_heading_weight, offroad_weight=rc.offroad_weight,
        offroad_lat_limit=rc.offroad_lat_limit, offroad_dist_limit=rc.offroad_dist_limit,
        idle_weight=rc.idle_weight, idle_speed=rc.idle_speed,
        ttc_vehicle_alpha=rc.ttc_vehicle_alpha, ttc_vehicle_pmax=rc.ttc_vehicle_pmax,
        ttc_edge_alpha=rc.ttc_edge_alpha, ttc_edge_pmax=rc.ttc_edge_pmax, ttc_floor=rc.ttc_floor,
        edge_range=rc.edge_range, crash_speed_limit=CRASH_SPEED_LIMIT, offstage_x=OFFSTAGE_X,
    )
    assert set(vals) == set(N.CONST_FIELDS)
    for name, v in vals.items():
        setattr(k, name, float(v))
    return k


def pack_scenes(scene_tables, type_norm: float, road_radius: float = 10.0,
                 agent_reach: float = 0.0, spatial_index: bool = True):
    """Concatenate per-scene blobs (layout documented in the C header).  The
    type feature is float32(type / type_norm), the reference's own cast.  The
    part the kernel copies to shared memory ends with the spatial-index header;
    the index's candidate lists follow it and stay in global memory."""
    blobs, meta, off = [], [], 0
    for t in scene_tables:
        P, KL, KE = t.num_segments, len(t.lane_index), len(t.edge_index)
        L, E = t.lane_index, t.edge_index
        parts = [np.ascontiguousarray(t.midpoints, dtype=np.float64),        # f64x2 mid[P]
                 np.ascontiguousarray(t.directions, dtype=np.float64),       # f64x2 dir[P]
                 np.ascontiguousarray(t.half_lengths, dtype=np.float64),
                 np.ascontiguousarray(t.half_widths, dtype=np.float64),
                 (t.type_codes.astype(np.float64) / type_norm).astype(np.float32),
                 np.ascontiguousarray(np.concatenate([t.midpoints[L], t.directions[L]], axis=1)),
                 np.ascontiguousarray(t.half_lengths[L], dtype=np.float64),
                 np.ascontiguousarray(t.midpoints[E], dtype=np.float64),
                 E.astype(np.int32)]
        chunk = bytearray()
        for a in parts:
            b = a.tobytes()
            chunk += b + bytes(_align16(len(b)) - len(b))
        edge_ext = float((t.half_lengths[t.edge_index] + t.half_widths[t.edge_index]).max()) \
            if len(t.edge_index) else 0.0
        head, aux = build_scene_index(t.midpoints, t.directions, t.half_lengths, t.half_widths,
                                      t.lane_index, t.edge_index, road_radius,
                                      agent_reach + edge_ext + 1e-6)
        if not spatial_index:
            head, aux = head[:32] + bytes(32), b""
        chunk += head
        smem_bytes = len(chunk)
        chunk += aux + bytes(_align16(len(aux)) - len(aux))
        blobs.append(bytes(chunk))
        meta.append([off, smem_bytes, P, KL, KE, off + smem_bytes, len(aux), 0])
        off += len(chunk)
    blob = np.frombuffer(b"".join(blobs), dtype=np.uint8).copy()
    max_bytes = max(m[1] for m in meta)
    max_p = max(m[2] for m in meta)
    return blob, np.asarray(meta, dtype=np.int64), max_bytes, max_p


def per_world_blobs(blob: np.ndarray, meta: np.ndarray, scene_of_world, grid_offsets):
    """Scenes whose blob exceeds shared memory (DgDims.geometry_global): one
    copy of the scene blob per world, appended after the shared per-scene
    blobs, with the segment / lane / edge midpoints already moved by the
    world's grid offset -- the same float64 ``mid + offset`` the kernel applies
    when it stages a blob in shared memory.  The spatial-index lists stay
    shared (meta[5] keeps pointing at the scene's copy)."""
    parts, wmeta, off = [blob.tobytes()], [], len(blob)
    for w, s in enumerate(np.asarray(scene_of_world)):
        o, nb, P, KL, KE, aux_off, aux_len, _ = (int(v) for v in meta[s])
        chunk = np.frombuffer(bytearray(blob[o:o + nb].tobytes()), dtype=np.uint8)
        ox, oy = float(grid_offsets[w][0]), float(grid_offsets[w][1])
        lane_at = 32 * P + _align16(8 * P) * 2 + _align16(4 * P)
        edge_at = lane_at + 32 * KL + _align16(8 * KL)
        mid = chunk[:16 * P].view(np.float64).reshape(P, 2)
        lane = chunk[lane_at:lane_at + 32 * KL].view(np.float64).reshape(KL, 4)
        edge = chunk[edge_at:edge_at + 16 * KE].view(np.float64).reshape(KE, 2)
        for a in (mid, lane, edge):
            a[:, 0] += ox
            a[:, 1] += oy
        parts.append(chunk.tobytes())
        wmeta.append([off, nb, P, KL, KE, aux_off, aux_len, 0])
        off += nb
    return np.frombuffer(b"".join(parts), dtype=np.uint8).copy(), np.asarray(wmeta, dtype=np.int64)


class _Lease:
    """numpy base object of one host slab hand-out: every array returned by a
    host step is a view of it, so it dies when the caller drops the last one."""
    __slots__ = ("__array_interface__", "__weakref__")


class HostSlabPool:
    """Pinned host slabs for the numpy step path, recycled once the caller has
    dropped every array of the step that filled them (weakref on the numpy
    base).  The reference returns fresh arrays each step (engine.py:307,
    397-406); a freed slab is exactly that without a cudaHostAlloc per step.
    Past ``max_pinned`` live slabs (a caller keeping every step's outputs)
    further slabs are pageable."""

    def __init__(self, nbytes: int, max_pinned: int = 16):
        self.nbytes = int(nbytes)
        self.max_pinned = int(max_pinned)
        self._slabs = []          # [pinned tensor, weakref to its current lease or None]

    def acquire(self):
        """(torch uint8 host tensor to copy into, numpy uint8 view of it)."""
        slot = next((s for s in self._slabs if s[1] is None or s[1]() is None), None)
        if slot is None:
            pinned = len(self._slabs) < self.max_pinned
            t = torch.empty(self.nbytes, dtype=torch.uint8, pin_memory=pinned)
            if not pinned:
                return t, t.numpy()
            slot = [t, None]
            self._slabs.append(slot)
        lease = _Lease()
        lease.__array_interface__ = {"data": (slot[0].data_ptr(), False), "shape": (self.nbytes,),
                                     "typestr": "|u1", "version": 3}
        slot[1] = weakref.ref(lease)
        return slot[0], np.asarray(lease)

    @property
    def pinned_slabs(self) -> int:
        return len(self._slabs)


class MappedSlabPool:
    """Mapped pinned host slabs (dg_host_alloc) the numpy step path hands out:
    the device writes the observation rows straight into the slab, only the
    non-zero prefix of each row's road / vehicle blocks crossing PCIe
    (dg_to_host), then DMAs the packed per-tick outputs behind them.  Each
    slab carries the per-row prefix lengths it holds (device int32 [rows][2])
    so a later step zeroes exactly what went stale.  Recycled like
    HostSlabPool; past ``max_slabs`` live slabs ``acquire`` returns None and
    the caller falls back to a full copy."""

    def __init__(self, lib, nbytes: int, rows: int, device, max_slabs: int = 8):
        self._lib = lib
        self.nbytes = int(nbytes)
        self.rows = int(rows)
        self.device = device
        self.max_slabs = int(max_slabs)
        self._slabs = []          # [host pointer, prev_len tensor, weakref to the current lease or None]

    def acquire(self):
        """(host pointer, prev_len device tensor, numpy uint8 view) or None."""
        slot = next((s for s in self._slabs if s[2] is None or s[2]() is None), None)
        if slot is None:
            if len(self._slabs) >= self.max_slabs:
                return None
            p = ct.c_void_p()
            N.check(self._lib, self._lib.dg_host_alloc(self.nbytes, ct.byref(p)), "dg_host_alloc")
            slot = [p.value, torch.zeros((self.rows, 2), dtype=torch.int32, device=self.device), None]
            self._slabs.append(slot)
        lease = _Lease()
        lease.__array_interface__ = {"data": (slot[0], False), "shape": (self.nbytes,), "typestr": "|u1",
                                     "version": 3}
        slot[2] = weakref.ref(lease)
        return slot[0], slot[1], np.asarray(lease)

    @property
    def slabs(self) -> int:
        return len(self._slabs)

    def release_all(self):
        """Free every slab (outstanding arrays of them become invalid)."""
        for ptr, _, _ in self._slabs:
            self._lib.dg_host_free(ct.c_void_p(ptr))
        self._slabs = []

    def __del__(self):
        try:
            self.release_all()
        except Exception:  # interpreter teardown
            pass


class StepOutput:
    """Result of one control tick (engine.py:70-76).  ``events`` and ``info``
    are built lazily from the packed output buffers."""

    def __init__(self, obs, rewards, dones, events4, info_src: dict, to_host: bool):
        self.obs = obs
        self.rewards = rewards
        self.dones = dones
        self._events4 = events4
        self._info_src = info_src
        self._host = to_host
        self._events = None
        self._info = None

    @property
    def events(self) -> dict:
        if self._events is None:
            self._events = {k: self._events4[..., i].astype(bool) if self._host
                            else self._events4[..., i].bool() for i, k in enumerate(EVENT_TYPES)}
        return self._events

    @property
    def info(self) -> dict:
        if self._info is None:
            s = self._info_src
            as_bool = (lambda a: a.astype(bool)) if self._host else (lambda a: a.bool())
            self._info = _LazyInfo({
                "alive": lambda: as_bool(s["alive"]),
                "alive_pre": lambda: as_bool(s["alive_pre"]),
                "state": lambda: {k: s["snapshot"][..., i, :, :] for i, k in enumerate(STATE_FIELDS)},
                "reason": lambda: s["reason"],
                "reward_terms": lambda: {k: s["terms"][..., i, :, :] for i, k in enumerate(TERM_NAMES)},
                "ttc_min": lambda: s["ttc_min"],
                "step": lambda: s["step"],
            })
        return self._info


class _LazyInfo(dict):
    """The step's info dict (engine.py:70-76 keys), each entry built on first
    access -- a loop that reads one entry per step (measure_engine's
    alive_pre, metrics.py:168-170) does not pay for the views of the others.
    Any whole-dict use (iteration, len, equality, copies) builds them all."""

    def __init__(self, makers: dict):
        super().__init__()
        self._makers = makers

    def __missing__(self, key):
        make = self._makers.get(key)
        if make is None:
            raise KeyError(key)
        v = make()
        dict.__setitem__(self, key, v)
        return v

    def _fill(self):
        for k in self._makers:
            if not dict.__contains__(self, k):
                self[k]
        return self

    def get(self, key, default=None):
        return self[key] if key in self._makers or dict.__contains__(self, key) else default

    def __contains__(self, key):
        return key in self._makers or dict.__contains__(self, key)

    def __iter__(self):
        return dict.__iter__(self._fill())

    def __len__(self):
        return dict.__len__(self._fill())

    def keys(self):
        return dict.keys(self._fill())

    def values(self):
        return dict.values(self._fill())

    def items(self):
        return dict.items(self._fill())

    def copy(self):
        return dict(self._fill().items())

    def __eq__(self, other):
        return dict.__eq__(self._fill(), other)

    __hash__ = None

    def __repr__(self):
        return dict.__repr__(self._fill())


@dataclass(eq=False)
class StepBuffers:
    """Preallocated device outputs for the zero-allocation path (bench,
    rollouts).  ``obs`` may be any [W][M][D] float32 view, e.g. one slot of
    a rollout ring."""

    obs: torch.Tensor
    aux: torch.Tensor
    views: dict
    # resident ring (new_rollout_buffers): per slot and agent the length of the road /
    # vehicle block prefix that can be non-zero; past it every float of the slot is
    # zero, so the step kernel clears only what a row's new content no longer covers
    # (DgStepIO.obs_resident).  The obs of a resident ring belong to the engine:
    # write them only through it (observe(out=slot) re-marks the slot).
    prefix: torch.Tensor | None = None

    def mark_dirty(self, slot: int | None = None) -> None:
        """The obs of ``slot`` (None: every slot) were written outside the
        engine's steps: the next step into it clears the whole blocks."""
        if self.prefix is not None:
            p = self.prefix if slot is None else self.prefix[slot]
            p[..., 0] = 0x7fff
            p[..., 1] = 0x7fff


class Engine:
    """Owner of the (W, M) agent state over a world batch, on one GPU.

    Performance knobs (results are identical under every setting):
    ``spatial_index`` (per-cell candidate lists vs full scans),
    ``warps_per_world`` / ``launch_mode`` (kernel shape, fused vs split), and
    ``geometry_global`` -- None stages each world's scene in shared memory
    (fused kernel) and falls back to per-world blobs read from global memory
    by the split kernels only for scenes too large for it; True / False force
    either path.
    """

    def __init__(self, worlds, scenes, assignment, frictions, config: SimConfig,
                 obs_config: ObsConfig | None = None, reward_config: RewardConfig | None = None,
                 params: VehicleParams | None = None, bicycle: BicycleParams | None = None,
                 device=None, spatial_index: bool = True, warps_per_world: int | None = None,
                 launch_mode: int | None = None, geometry_global: bool | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("drivegrid-b200 Engine needs a CUDA device (no CPU fallback)")
        self._lib = N.load_library()
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.config = config
        self.obs_config = obs_config or ObsConfig()
        self.reward_config = reward_config or RewardConfig()
        self.params = params or VehicleParams()
        self.bicycle = bicycle or BicycleParams()
        self.worlds = worlds
        self.frictions = frictions
        if isinstance(worlds, DeviceWorldBatch):
            # on-device world construction: the spawn table and initial state are
            # written by the GPU into the arrays the engine binds (worldgen.py)
            t = device_engine_tables(worlds, frictions, config, self.params)
        else:
            t = build_tables(worlds, scenes, assignment, frictions, config, self.params)
        self.tables = t
        built = getattr(t, "dev", None)
        W, M = t.W, t.M
        self.W, self.M = W, M
        self.valid = t.valid.copy()
        self.length, self.width = t.length, t.width
        self.r_hull, self.d_hull = t.r_hull, t.d_hull
        self.mu_eff, self.weather = t.mu_eff, t.weather
        self._lane = None
        self._edge = None

        dev = self.device

        def up(a, dtype, key=None):
            if built is not None and key in built:
                return built[key]
            return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(dev)

        reach = float((t.r_hull + t.d_hull).max())
        blob, meta, max_bytes, max_p = pack_scenes(t.scenes, self.obs_config.type_norm,
                                                   self.obs_config.road_radius, reach,
                                                   spatial_index=spatial_index)
        self._d = d = {
            "scene_blob": up(blob, torch.uint8),
            "scene_meta": up(meta, torch.int64),
            "scene_of_world": up(t.scene_of_world, torch.int32, "assignment"),
            "grid_offset": up(t.grid_offsets, torch.float64, "grid_offset"),
            "mu_eff": up(t.mu_eff, torch.float64),
            "weather": up(t.weather, torch.float64),
            "valid": up(t.valid, torch.uint8, "valid"),
            "length": up(t.length, torch.float64, "length"),
            "width": up(t.width, torch.float64, "width"),
            "r_hull": up(t.r_hull, torch.float64, "r_hull"),
            "d_hull": up(t.d_hull, torch.float64, "d_hull"),
            "state": up(None if built is not None else np.stack([t.state0[k] for k in STATE_FIELDS]),
                        torch.float64, "state"),
            "alive": up(t.valid, torch.uint8, "alive"),
            "reason": torch.zeros((W, M), dtype=torch.int8, device=dev),
            "event_seen": torch.zeros((W, M), dtype=torch.uint8, device=dev),
            "spawn_step": torch.zeros((W, M), dtype=torch.int32, device=dev),
            "step_count": torch.zeros((W,), dtype=torch.int32, device=dev),
            "start_xy": up(None if built is not None else t.start_xy, torch.float64, "start_xy"),
            "goal_xy": up(None if built is not None else t.goal_xy, torch.float64, "goal_xy"),
            "start_yaw": up(None if built is not None else t.start_yaw, torch.float64, "start_yaw"),
            "error_word": torch.full((1,), N.DG_NO_ERROR, dtype=torch.int32, device=dev),
            # zeroed once: the split kernels copy whole AgentRec records, padding included
            "scratch": torch.zeros(int(self._lib.dg_scratch_bytes(W, M)), dtype=torch.uint8, device=dev),
        }
        oc = self.obs_config
        dims = N.DgDims(W=W, M=M, obs_dim=oc.obs_dim, ego_dim=oc.ego_dim, k_road=oc.k_road,
                        k_vehicles=oc.k_vehicles, include_weather=int(oc.include_weather),
                        dynamic=int(config.dynamics_mode == "dynamic"), decimation=config.decimation,
                        episode_len=config.episode_len, invincible=int(config.invincible),
                        collision_warmup=self.reward_config.collision_warmup_steps,
                        num_scenes=len(t.scenes), max_scene_bytes=max_bytes, max_segments=max_p)
        desc = N.DgEngineDesc(dims=dims, k=make_consts(config, oc, self.reward_config, self.params,
                                                       self.bicycle))
        for name in ("scene_blob", "scene_meta", "scene_of_world", "grid_offset", "mu_eff", "weather",
                     "valid", "length", "width", "r_hull", "d_hull", "state", "alive", "reason",
                     "event_seen", "spawn_step", "step_count", "start_xy", "goal_xy", "start_yaw",
                     "error_word", "scratch"):
            setattr(desc, name, d[name].data_ptr())
        handle = ct.c_void_p()
        status = self._lib.dg_create(ct.byref(desc), ct.byref(handle)) if not geometry_global else N.DG_ENOSUPPORT
        too_big = status == N.DG_ENOSUPPORT and b"shared memory" in (self._lib.dg_last_error() or b"")
        if geometry_global or (too_big and geometry_global is None):
            # a scene too large to stage in shared memory: per-world translated
            # blobs read from global memory instead
            wblob, wmeta = per_world_blobs(blob, meta, t.scene_of_world, t.grid_offsets)
            d["scene_blob"], d["scene_meta"] = up(wblob, torch.uint8), up(wmeta, torch.int64)
            d["scene_of_world"] = up(np.arange(W), torch.int32)
            desc.dims.num_scenes, desc.dims.geometry_global = W, 1
            for name in ("scene_blob", "scene_meta", "scene_of_world"):
                setattr(desc, name, d[name].data_ptr())
            status = self._lib.dg_create(ct.byref(desc), ct.byref(handle))
        N.check(self._lib, status, "dg_create")
        self.geometry_global = bool(desc.dims.geometry_global)
        self._h = handle
        self._desc = desc
        if self.geometry_global and launch_mode in (0, 2):
            # global-memory geometry on the fused kernel's kGeoGlobal variants
            # (multi-tick launches): 4 warps x 4 CTAs/SM, or mode 2
            if launch_mode == 2:
                self.tune(min(M, 7), 0, mode=2)
            else:
                self.tune(warps_per_world or min(M, 4), 4 if M > 4 else 0)
        elif self.geometry_global:
            # global-memory geometry: the split kernels, one warp per agent (2x the
            # fused variant on the dense 6,000-segment scene, tools/dense_scene_timing.py)
            self.tune(warps_per_world if warps_per_world in (2, 4, 8) else 4, 0, mode=1)
        elif launch_mode == 1:
            self.tune(warps_per_world or 4, 0, mode=1)
        elif warps_per_world:
            self.tune(warps_per_world, 0, mode=launch_mode or 0)
        elif W > 2 * torch.cuda.get_device_properties(self.device).multi_processor_count:
            # more worlds than 8-warp CTAs fit at once (2 per SM): 4 warps/world,
            # 4 CTAs/SM (measured on B200: 512 worlds 270 -> 307 M CASPS, 1024: 280 -> 317)
            self.tune(min(M, 4), 4 if M > 4 else 0)
        else:
            # every world resident as an 8-warp CTA (2 per SM): latency-bound regime;
            # mode 2: 7 scan warps + a warp running the next tick's physics meanwhile
            mode = 2 if launch_mode is None else launch_mode
            self.tune(min(M, 7 if mode == 2 else 8), 0, mode=mode)
        self._step_count = 0
        self.phase_seconds = {k: 0.0 for k in PHASES}
        self._act_dev = torch.empty((W, M, 3), dtype=torch.float64, device=dev)
        self._act_host = torch.empty((W, M, 3), dtype=torch.float64).pin_memory()
        # host-path outputs in ONE device allocation [obs | pad | aux] -> one D2H copy per step
        obs_bytes = W * M * oc.obs_dim * 4
        self._host_obs_bytes = _align16(obs_bytes)
        _, aux_total = self._aux_layout()
        # [obs | aux | 5 x int64 phase cycles]: the phase counters ride in the same
        # D2H as the per-tick outputs
        self._phase_off = self._host_obs_bytes + aux_total
        self._host_blob = torch.zeros(self._phase_off + 48, dtype=torch.uint8, device=dev)
        self._obs_dev = self._host_blob[:obs_bytes].view(torch.float32).view(W, M, oc.obs_dim)
        aux_dev = self._host_blob[self._host_obs_bytes:self._phase_off]
        self._host_bufs = StepBuffers(self._obs_dev, aux_dev, self._views(aux_dev))
        self._host_pool = HostSlabPool(self._host_blob.numel())
        self._mapped_pool = MappedSlabPool(self._lib, self._host_blob.numel(), W * M, dev)
        self.d2h_bytes = torch.zeros(1, dtype=torch.int64, device=dev)   # obs bytes written by dg_to_host
        self._prefix_dev = torch.zeros((W, M, 2), dtype=torch.int16, device=dev)   # non-zero obs prefixes
        self._resident = weakref.WeakSet()     # resident rollout rings of this engine
        # per-phase device cycles of the host-path steps (DgStepIO.phase_cycles)
        self._phase_dev = self._host_blob[self._phase_off:self._phase_off + 40].view(torch.int64)
        self._phase_host = None          # int64 [5] view of the last host slab
        self._phase_prev = np.zeros(5, dtype=np.int64)
        self.launches = 0
        self._metrics_on = False
        self._host_lay = None
        self._host_io = {}
        self._drac_max = None
        self._metric_seen = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.dg_destroy(h)
            except Exception:  # interpreter teardown
                pass
            self._h = None

    # ------------------------------------------------------------------ buffers
    def _stream(self):
        return ct.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _aux_layout(self, slots: int | None = None):
        W, M = self.W, self.M
        WM = W * M
        lay, off = {}, 0
        k = 1 if slots is None else int(slots)
        lead = () if slots is None else (k,)
        for name, nbytes, dtype, shape in (
                ("rewards", 8 * WM, torch.float64, (W, M)),
                ("ttc_min", 8 * WM, torch.float64, (W, M)),
                ("terms", 8 * 7 * WM, torch.float64, (7, W, M)),
                ("snapshot", 8 * 12 * WM, torch.float64, (12, W, M)),
                ("events", 4 * WM, torch.uint8, (W, M, 4)),
                ("dones", WM, torch.uint8, (W, M)),
                ("reason", WM, torch.int8, (W, M)),
                ("alive", WM, torch.uint8, (W, M)),
                ("alive_pre", WM, torch.uint8, (W, M))):
            lay[name] = (off, k * nbytes, dtype, lead + shape)
            off = _align16(off + k * nbytes)
        return lay, off

    def _host_views(self, aux: np.ndarray) -> dict:
        """numpy views of a host copy of the packed aux buffer (one tick)."""
        lay = self._host_lay
        if lay is None:
            lay = self._host_lay = [(name, o, n, torch.empty((), dtype=dt).numpy().dtype, shape)
                                    for name, (o, n, dt, shape) in self._aux_layout()[0].items()]
        # each field's view is made on first access (a step reads rewards / dones /
        # events; info entries only when asked for)
        return _LazyInfo({name: (lambda o=o, n=n, dt=dt, shape=shape: aux[o:o + n].view(dt).reshape(shape))
                          for name, o, n, dt, shape in lay})

    def _views(self, aux: torch.Tensor, slots: int | None = None) -> dict:
        lay, _ = self._aux_layout(slots)
        return {name: aux[o:o + n].view(dt).view(shape) for name, (o, n, dt, shape) in lay.items()}

    def _new_buffers(self, obs: torch.Tensor | None = None) -> StepBuffers:
        _, total = self._aux_layout()
        aux = torch.zeros(total, dtype=torch.uint8, device=self.device)   # padding defined (initcheck)
        if obs is None:
            obs = torch.empty((self.W, self.M, self.obs_config.obs_dim), dtype=torch.float32,
                              device=self.device)
        return StepBuffers(obs, aux, self._views(aux))

    def new_step_buffers(self, obs: torch.Tensor | None = None) -> StepBuffers:
        return self._new_buffers(obs)

    def new_rollout_buffers(self, slots: int, resident: bool | None = None) -> StepBuffers:
        """Ring of ``slots`` per-tick outputs for ``launch_step(ticks=...)``:
        obs [S][W][M][D] and every aux view with a leading slot axis.  A
        resident ring (zeroed once, with its prefix record) lets every later
        step clear only the spans of its rows that the new content no longer
        covers instead of the whole 7.7 KB row."""
        if resident is None:
            resident = os.environ.get("DG_RESIDENT", "1") != "0"
        _, total = self._aux_layout(slots)
        aux = torch.zeros(total, dtype=torch.uint8, device=self.device)   # padding defined (initcheck)
        shape = (slots, self.W, self.M, self.obs_config.obs_dim)
        if resident:
            obs = torch.zeros(shape, dtype=torch.float32, device=self.device)
            prefix = torch.zeros((slots, self.W, self.M, 2), dtype=torch.int16, device=self.device)
            bufs = StepBuffers(obs, aux, self._views(aux, slots), prefix)
            self._resident.add(bufs)
            return bufs
        obs = torch.empty(shape, dtype=torch.float32, device=self.device)
        return StepBuffers(obs, aux, self._views(aux, slots))

    def launch_shape(self) -> dict:
        return dict(self._shape)

    @property
    def index_stride(self) -> int:
        """int32 entries per agent of the ``index_out`` debug record."""
        return int(self._lib.dg_index_stride(self._h))

    def new_index_buffer(self, slots: int = 1) -> torch.Tensor:
        """[slots][W][M][index_stride] int32, filled with -1."""
        return torch.full((int(slots), self.W, self.M, self.index_stride), -1, dtype=torch.int32,
                          device=self.device)

    def tune(self, warps_per_world: int, ctas_per_sm: int = 0, mode: int = 0) -> None:
        """Launch shape knob; results are unaffected.  mode 0: fused world
        kernel with ``warps_per_world`` warps; mode 1: split physics + per-agent
        kernels with ``warps_per_world`` agents per CTA; mode 2: fused with one
        more warp that computes tick t + 1's physics while the others scan tick t.  ``ctas_per_sm`` picks
        the register budget of the kernel variant (0 = default)."""
        N.check(self._lib, self._lib.dg_tune(self._h, int(mode), int(warps_per_world), int(ctas_per_sm)),
                "dg_tune")
        self._shape = {"mode": ("fused", "split", "fused+physics-warp")[int(mode)], "warps": int(warps_per_world),
                       "ctas_per_sm": int(ctas_per_sm)}

    # ------------------------------------------------------------------ device state views
    @property
    def state_tensor(self) -> torch.Tensor:
        """[12][W][M] float64 device tensor (live, not a copy)."""
        return self._d["state"]

    def device_tables(self) -> dict:
        return self._d

    @property
    def step_count(self) -> int:
        return self._step_count

    @step_count.setter
    def step_count(self, value: int):
        N.check(self._lib, self._lib.dg_set_step_count(self._h, int(value), self._stream()),
                "dg_set_step_count")
        self._step_count = int(value)

    def _host(self, name):
        return self._d[name].cpu().numpy()

    @property
    def state(self) -> dict:
        st = torch.empty(self._d["state"].shape, dtype=torch.float64, pin_memory=True)
        N.check(self._lib, self._lib.dg_get_state(self._h, st.data_ptr(), self._stream()), "dg_get_state")
        torch.cuda.current_stream(self.device).synchronize()
        st = st.numpy()
        return {k: st[i].copy() for i, k in enumerate(STATE_FIELDS)}

    def load_state_tensor(self, state: torch.Tensor) -> None:
        """Replace the whole [12][W][M] float64 state (device or host tensor) via dg_set_state."""
        if tuple(state.shape) != tuple(self._d["state"].shape) or state.dtype != torch.float64:
            raise ValueError(f"state must be float64 {tuple(self._d['state'].shape)}")
        state = state.contiguous()
        N.check(self._lib, self._lib.dg_set_state(self._h, state.data_ptr(), self._stream()), "dg_set_state")
        if not state.is_cuda:
            torch.cuda.current_stream(self.device).synchronize()

    def set_state(self, values: dict) -> None:
        """Overwrite state fields (host or device arrays, global coordinates)."""
        for k, v in values.items():
            i = STATE_FIELDS.index(k)
            self._d["state"][i].copy_(torch.as_tensor(np.asarray(v, dtype=np.float64)
                                                      if not isinstance(v, torch.Tensor) else v))

    @property
    def alive(self) -> np.ndarray:
        return self._host("alive").astype(bool)

    @alive.setter
    def alive(self, value):
        self._d["alive"].copy_(torch.as_tensor(np.asarray(value, dtype=np.uint8)))

    @property
    def reason(self) -> np.ndarray:
        return self._host("reason")

    @property
    def spawn_step(self) -> np.ndarray:
        return self._host("spawn_step").astype(np.int64)

    @property
    def start_xy(self) -> np.ndarray:
        return self._host("start_xy")

    @property
    def goal_xy(self) -> np.ndarray:
        return self._host("goal_xy")

    @property
    def start_yaw(self) -> np.ndarray:
        return self._host("start_yaw")

    def set_goals(self, goal_xy) -> None:
        self._d["goal_xy"].copy_(torch.as_tensor(np.asarray(goal_xy, dtype=np.float64)))

    @property
    def event_seen(self) -> dict:
        bits = self._host("event_seen")
        return {k: (bits >> i & 1).astype(bool) for i, k in enumerate(EVENT_TYPES)}

    @property
    def pos(self) -> np.ndarray:
        st = self.state
        return np.stack([st["x"], st["y"]], axis=-1)

    @property
    def lane(self) -> dict:
        if self._lane is None:
            self._lane = (self.worlds.compact_subset("lane") if isinstance(self.worlds, DeviceWorldBatch) else
                          compact_subset(self.worlds, lane_mask_of(self.worlds.type_codes, self.worlds.mask)))
        return self._lane

    @property
    def edge(self) -> dict:
        if self._edge is None:
            self._edge = (self.worlds.compact_subset("edge") if isinstance(self.worlds, DeviceWorldBatch) else
                          compact_subset(self.worlds, edge_mask_of(self.worlds.type_codes, self.worlds.mask)))
        return self._edge

    def reset_phase_timers(self):
        self.phase_seconds = {k: 0.0 for k in PHASES}

    # ------------------------------------------------------------------ errors
    def _raise_nonfinite(self, flat: int):
        w, m = (flat // (3 * self.M)) % self.W, (flat // 3) % self.M
        raise ValueError(f"non-finite action for world {w} agent {m}")

    def check_actions(self, actions: torch.Tensor) -> None:
        """Device finiteness scan + one sync; raises exactly like the reference."""
        N.check(self._lib, self._lib.dg_check_actions(self._h, _ptr(actions),
                                                      int(actions.dtype == torch.float64),
                                                      self._stream()), "dg_check_actions")
        self.raise_pending_error()

    def raise_pending_error(self) -> None:
        flat = ct.c_int32(-1)
        N.check(self._lib, self._lib.dg_read_error(self._h, ct.byref(flat), self._stream()),
                "dg_read_error")
        if flat.value >= 0:
            # a rejected tick stops its world where it was (a multi-tick launch
            # may have advanced the others): the host counter follows the device
            self._step_count = int(self._d["step_count"].min().item())
            self._raise_nonfinite(flat.value)

    # ------------------------------------------------------------------ observe
    def observe(self, ttc_min: torch.Tensor | None = None, out: torch.Tensor | None = None,
                as_numpy: bool = True, next_actions: torch.Tensor | None = None, steer_gain: float = 2.0,
                throttle: float = 0.5):
        """Observation of the current state (engine.py:297-300); with
        ``next_actions`` the LaneFollower actions for it are fused in."""
        obs = out if out is not None else torch.empty_like(self._obs_dev)
        if out is not None:
            self._mark_written(out)
        N.check(self._lib, self._lib.dg_observe(self._h, _ptr(obs), _ptr(ttc_min), _ptr(next_actions),
                                                float(steer_gain), float(throttle), self._stream()),
                "dg_observe")
        self.launches += 1
        if as_numpy:
            return obs.cpu().numpy()
        return obs

    def _mark_written(self, out: torch.Tensor) -> None:
        """``out`` is about to be written outside a step: a resident ring slot it
        lies in loses its prefix record."""
        lo, hi = out.data_ptr(), out.data_ptr() + out.numel() * out.element_size()
        for b in list(self._resident):
            base = b.obs.data_ptr()
            per = b.obs[0].numel() * b.obs.element_size()
            end = base + per * b.obs.shape[0]
            if lo < end and hi > base:
                first, last = max(lo - base, 0) // per, (min(hi, end) - base - 1) // per
                b.prefix[first:last + 1] = 0x7fff

    def observe_device(self, out: torch.Tensor | None = None) -> torch.Tensor:
        return self.observe(out=out, as_numpy=False)

    # ------------------------------------------------------------------ step
    def launch_step(self, actions: torch.Tensor, bufs: StepBuffers, autoreset: bool = False,
                    snapshot: bool = True, terms: bool = True, next_actions: torch.Tensor | None = None,
                    steer_gain: float = 2.0, throttle: float = 0.5,
                    event_counts: torch.Tensor | None = None, ticks: int = 1, ring_start: int = 0,
                    drac_max: torch.Tensor | None = None, metric_seen: torch.Tensor | None = None,
                    index_out: torch.Tensor | None = None, prefix_out: torch.Tensor | None = None) -> None:
        """Enqueue one fused launch on the current stream; no sync, no checks
        beyond the device-side non-finite guard.  Used by the fast paths.
        ``next_actions`` (float64 [W][M][3], may alias ``actions``) receives
        the fused LaneFollower's actions on the last tick's observation;
        ``event_counts`` (int32 [W][5]) accumulates per-world goal / collision /
        crash / lane_forbidden events and alive agent-ticks on the device.

        ``ticks`` > 1 runs that many control ticks in the same launch (each
        world's CTA keeps its scene and agents in shared memory across them):
        tick t reads ``actions[t]`` ([T][W][M][3]) -- or, with ``next_actions``,
        ``actions`` ([W][M][3]) at tick 0 and the fused policy's actions after
        -- and writes slot ``(ring_start + t) % S`` of rollout buffers with S
        slots (``new_rollout_buffers``).

        ``drac_max`` (float64 [W][M]) / ``metric_seen`` (uint8 [W][M]) are the
        in-kernel episode-metric accumulators (default: the engine's own when
        ``track_episode_metrics`` is on).  ``index_out`` (int32 [S][W][M][
        ``index_stride``], S = ring slots) receives the integer decisions of
        every tick: nearest-lane index, road slot -> segment map, neighbour
        order (layout: ``DgStepIO.index_out`` in the C header).  ``prefix_out``
        (int16 [S][W][M][2]) receives per agent the length of the road / vehicle
        block prefix that can be non-zero (``DgStepIO.prefix_out``)."""
        resident = prefix_out is None and bufs.prefix is not None
        if resident:
            prefix_out = bufs.prefix
        if self._shape["mode"] == "split" and (ticks > 1 or bufs.obs.dim() == 4):
            # the split kernels take one tick per launch and write one output
            # set: tick t goes to ring slot (ring_start + t) % S through views
            slots = bufs.obs.shape[0] if bufs.obs.dim() == 4 else 1
            for t in range(int(ticks)):
                if next_actions is not None:
                    a_t = actions if t == 0 else next_actions
                else:
                    a_t = actions[t] if ticks > 1 or actions.dim() == 4 else actions
                slot = (ring_start + t) % slots
                one = bufs if bufs.obs.dim() == 3 else StepBuffers(
                    bufs.obs[slot], bufs.aux, {k: v[slot] for k, v in bufs.views.items()})
                self.launch_step(a_t, one, autoreset, snapshot, terms, next_actions, steer_gain, throttle,
                                 event_counts, 1, 0, drac_max, metric_seen,
                                 None if index_out is None else index_out.view(-1, *index_out.shape[-3:])[slot],
                                 None if prefix_out is None else prefix_out.view(-1, self.W, self.M, 2)[slot])
            return
        if prefix_out is not None and (prefix_out.dtype != torch.int16 or not prefix_out.is_contiguous()
                                       or prefix_out.numel() % (self.W * self.M * 2)):
            raise ValueError("prefix_out must be a contiguous int16 CUDA tensor of [S][W][M][2]")
        io = self._step_io(actions, bufs, autoreset, snapshot, terms, next_actions, steer_gain, throttle,
                           event_counts, ticks, ring_start, drac_max, metric_seen, index_out, prefix_out, resident)
        N.check(self._lib, self._lib.dg_step(self._h, ct.byref(io), self._stream()), "dg_step")
        self._step_count += int(ticks)
        self.launches += 1

    def _step_io(self, actions, bufs, autoreset=False, snapshot=True, terms=True, next_actions=None,
                 steer_gain=2.0, throttle=0.5, event_counts=None, ticks=1, ring_start=0, drac_max=None,
                 metric_seen=None, index_out=None, prefix_out=None, resident=False, phase_cycles=None):
        if self._metrics_on:
            drac_max = self._drac_max if drac_max is None else drac_max
            metric_seen = self._metric_seen if metric_seen is None else metric_seen
        v = bufs.views
        slots = bufs.obs.shape[0] if bufs.obs.dim() == 4 else 1
        io = N.DgStepIO(actions=actions.data_ptr(), actions_f64=int(actions.dtype == torch.float64),
                        autoreset=int(autoreset), obs=bufs.obs.data_ptr(),
                        rewards=v["rewards"].data_ptr(), dones=v["dones"].data_ptr(),
                        events=v["events"].data_ptr(), reason_out=v["reason"].data_ptr(),
                        alive_out=v["alive"].data_ptr(), alive_pre_out=v["alive_pre"].data_ptr(),
                        ttc_min_out=v["ttc_min"].data_ptr(),
                        terms_out=v["terms"].data_ptr() if terms else None,
                        snapshot_out=v["snapshot"].data_ptr() if snapshot else None,
                        next_actions=next_actions.data_ptr() if next_actions is not None else None,
                        policy_gain=float(steer_gain), policy_throttle=float(throttle),
                        event_counts=event_counts.data_ptr() if event_counts is not None else None,
                        ticks=int(ticks), ring_slots=int(slots), ring_start=int(ring_start),
                        drac_max=_ptr(drac_max), metric_seen=_ptr(metric_seen), index_out=_ptr(index_out),
                        prefix_out=_ptr(prefix_out), obs_resident=int(bool(resident)),
                        phase_cycles=_ptr(phase_cycles))
        if index_out is not None:
            want = (slots, self.W, self.M, self.index_stride)
            if (index_out.dtype != torch.int32 or not index_out.is_cuda or not index_out.is_contiguous()
                    or index_out.numel() != int(np.prod(want))):
                raise ValueError(f"index_out must be a contiguous int32 CUDA tensor of {want} elements")
        return io

    def rollout(self, actions, ticks: int | None = None, autoreset: bool = False, policy=None,
                steer_gain: float = 2.0, throttle: float = 0.5, bufs: StepBuffers | None = None,
                next_actions: torch.Tensor | None = None, values: torch.Tensor | None = None,
                sample: bool = False, seed: int = 0, counter0: int = 0, log_probs: torch.Tensor | None = None,
                actions_out: torch.Tensor | None = None) -> StepOutput:
        """T control ticks in ONE kernel launch -- the same results as T
        ``step`` calls (env.py:48-65 in a loop).

        ``actions``: a [T][W][M][3] stream replayed tick by tick, or with
        ``policy="lane_follower"`` the [W][M][3] actions of the first tick,
        the fused LaneFollower (policies.py:21-43) driving every later tick
        from that tick's observation (``ticks`` required).  A replayed stream
        is validated before anything runs and raises like ``step``.  Returns a
        device StepOutput whose arrays carry a leading tick axis; the policy's
        actions for the tick after the last are in ``next_actions``.

        ``policy`` may also be a ``PolicyMLP`` (BASELINE configs[4]): every
        tick is one step launch followed by the policy forward on that tick's
        observation (two tcgen05 launches), whose actor mean is the next
        tick's action -- the whole loop stays on the device and is CUDA-graph
        capturable.  ``values`` ([T][W][M] float32) receives the critic's
        value of each tick's observation; with ``sample`` the actions are PPO
        draws (Philox, ``seed``, counter ``counter0 + t``) recorded in
        ``actions_out`` ([T][W][M][3] f32) with their ``log_probs``."""
        if policy is not None and not isinstance(policy, str):
            return self._rollout_mlp(actions, ticks, autoreset, policy, bufs, next_actions, values,
                                     dict(sample=sample, seed=seed, counter0=counter0, log_probs=log_probs,
                                          actions_out=actions_out))
        dev = self.device
        a = actions if isinstance(actions, torch.Tensor) else torch.as_tensor(np.asarray(actions, np.float64))
        if a.dtype not in (torch.float32, torch.float64):
            a = a.to(torch.float64)
        a = a.to(dev).contiguous()
        if policy is None:
            if a.dim() != 4 or tuple(a.shape[1:]) != (self.W, self.M, 3):
                raise ValueError(f"actions shape {tuple(a.shape)}, expected (T, {self.W}, {self.M}, 3)")
            T = a.shape[0] if ticks is None else int(ticks)
            if T > a.shape[0]:
                raise ValueError(f"{T} ticks but only {a.shape[0]} action frames")
            bad = ~torch.isfinite(a[:T])
            if bool(bad.any()):
                t, w, m, _ = (int(i) for i in bad.nonzero()[0])
                raise ValueError(f"non-finite action for world {w} agent {m}")
        elif policy == "lane_follower":
            if tuple(a.shape) != (self.W, self.M, 3):
                raise ValueError(f"actions shape {tuple(a.shape)}, expected {(self.W, self.M, 3)}")
            if ticks is None:
                raise ValueError("rollout with a policy needs ticks")
            T = int(ticks)
            self.check_actions(a)
            if next_actions is None:
                next_actions = torch.empty((self.W, self.M, 3), dtype=torch.float64, device=dev)
        else:
            raise ValueError(f"unknown rollout policy {policy!r}")
        if T < 1:
            raise ValueError("ticks must be >= 1")
        if bufs is None:
            bufs = self.new_rollout_buffers(T)
        self.launch_step(a, bufs, autoreset=autoreset, ticks=T,
                         next_actions=next_actions if policy else None,
                         steer_gain=steer_gain, throttle=throttle)
        self.raise_pending_error()
        v = bufs.views
        src = dict(v)
        src["step"] = self._step_count
        out = StepOutput(bufs.obs, v["rewards"], v["dones"].bool(), v["events"], src, to_host=False)
        out.next_actions = next_actions
        return out

    def _rollout_mlp(self, actions, ticks, autoreset, policy, bufs, next_actions, values, ppo) -> StepOutput:
        dev = self.device
        a = actions if isinstance(actions, torch.Tensor) else torch.as_tensor(np.asarray(actions, np.float64))
        a = a.to(device=dev, dtype=torch.float64).contiguous()
        if tuple(a.shape) != (self.W, self.M, 3):
            raise ValueError(f"actions shape {tuple(a.shape)}, expected {(self.W, self.M, 3)}")
        if ticks is None or int(ticks) < 1:
            raise ValueError("rollout with a policy needs ticks >= 1")
        T = int(ticks)
        self.check_actions(a)
        if bufs is None:
            bufs = self.new_rollout_buffers(T)
        slots = bufs.obs.shape[0] if bufs.obs.dim() == 4 else 1
        if values is not None and tuple(values.shape) != (T, self.W, self.M):
            raise ValueError(f"values shape {tuple(values.shape)}, expected {(T, self.W, self.M)}")
        acts = next_actions if next_actions is not None else torch.empty_like(a)
        if acts.data_ptr() != a.data_ptr():
            acts.copy_(a)
        for name, shape in (("log_probs", (T, self.W, self.M)), ("actions_out", (T, self.W, self.M, 3))):
            if ppo[name] is not None and tuple(ppo[name].shape) != shape:
                raise ValueError(f"{name} shape {tuple(ppo[name].shape)}, expected {shape}")
        self.run_mlp_ticks(acts, bufs, policy, T, autoreset=autoreset, values=values, **ppo)
        self.raise_pending_error()
        v = bufs.views
        src = dict(v)
        src["step"] = self._step_count
        out = StepOutput(bufs.obs, v["rewards"], v["dones"].bool(), v["events"], src, to_host=False)
        out.next_actions = acts
        return out

    def run_mlp_ticks(self, acts: torch.Tensor, bufs: StepBuffers, policy, ticks: int, ring_start: int = 0,
                      autoreset: bool = False, values: torch.Tensor | None = None,
                      event_counts: torch.Tensor | None = None, sample: bool = False, seed: int = 0,
                      counter0: int = 0, log_probs: torch.Tensor | None = None,
                      actions_out: torch.Tensor | None = None, overlap_critic: bool = True) -> None:
        """Enqueue ``ticks`` x (step launch -> policy forward): tick t reads
        ``acts`` ([W][M][3] float64) and the policy overwrites it with the next
        tick's actions (the mean, or a Philox draw with ``sample``, counter
        ``counter0 + t``); per tick t: ``values[t]``, ``log_probs[t]``,
        ``actions_out[t]`` (the action chosen on tick t's observation).  No
        sync, no checks (the fast path of ``rollout`` and the bench).

        With ``overlap_critic`` the value head -- which no later tick depends on
        -- runs on a side stream, so only step -> actor forward is on the
        rollout's critical path; the side stream joins the current one before
        this returns (also under CUDA-graph capture), and a ring slot is not
        overwritten before the critic has read it."""
        slots = bufs.obs.shape[0] if bufs.obs.dim() == 4 else 1
        side = None
        if values is not None and overlap_critic:
            side = self._side_stream()
            main = torch.cuda.current_stream(self.device)
            side.wait_stream(main)
            done = [None] * int(ticks)          # critic of tick t has read its slot
        for t in range(int(ticks)):
            slot = (ring_start + t) % slots
            if side is not None and t >= slots and done[t - slots] is not None:
                main.wait_event(done[t - slots])   # the step below overwrites the slot of tick t - slots
            self.launch_step(acts, bufs, autoreset=autoreset, ticks=1, ring_start=slot,
                             event_counts=event_counts)
            obs = bufs.obs[slot] if bufs.obs.dim() == 4 else bufs.obs
            pre = None
            if bufs.prefix is not None:   # the step just wrote this slot's valid-slot prefixes
                pre = bufs.prefix[slot] if bufs.prefix.dim() == 4 else bufs.prefix
            if side is not None:
                ready = torch.cuda.Event()
                ready.record(main)
            policy.forward(obs, actions=acts, value=None if values is None or side is not None else values[t],
                           sample=sample, prefix=pre, seed=seed, counter=counter0 + t,
                           log_prob=None if log_probs is None else log_probs[t],
                           actions_f32=None if actions_out is None else actions_out[t],
                           nets="actor" if side is not None else "both")
            self.launches += policy.launches()
            if side is not None:
                side.wait_event(ready)
                with torch.cuda.stream(side):
                    policy.forward(obs, value=values[t], prefix=pre, nets="critic")
                    done[t] = torch.cuda.Event()
                    done[t].record(side)
                self.launches += policy.launches()
        if side is not None:
            torch.cuda.current_stream(self.device).wait_stream(side)

    def _side_stream(self) -> torch.cuda.Stream:
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device)
        return self._side

    def step(self, actions, autoreset: bool = False) -> StepOutput:
        """One 30 Hz control tick (engine.py:334-406)."""
        if isinstance(actions, torch.Tensor) and actions.is_cuda:
            return self._step_device(actions, autoreset)
        return self._step_host(actions, autoreset)

    def _step_device(self, actions: torch.Tensor, autoreset: bool, check: bool = True) -> StepOutput:
        want = (self.W, self.M, 3)
        if tuple(actions.shape) != want:
            raise ValueError(f"actions shape {tuple(actions.shape)}, expected {want}")
        if actions.dtype not in (torch.float32, torch.float64):
            actions = actions.to(torch.float64)
        actions = actions.contiguous()
        if check:
            self.check_actions(actions)
        bufs = self._new_buffers()
        self.launch_step(actions, bufs, autoreset=autoreset)
        v = bufs.views
        src = dict(v)
        src["step"] = self._step_count
        return StepOutput(bufs.obs, v["rewards"], v["dones"].bool(), v["events"], src, to_host=False)

    def _book_phases(self, wall: float) -> None:
        """Split a step's device + delivery wall time over the reference's
        PHASES (engine.py:33, 342-395) in proportion to the device cycles the
        fused kernel spent in each (DgStepIO.phase_cycles); the split kernels do
        not record them -- their time goes to "physics"."""
        cyc = np.array(self._phase_host, dtype=np.int64)
        d = cyc - self._phase_prev
        self._phase_prev = cyc
        tot = float(d.sum())
        if tot <= 0.0:
            self.phase_seconds["physics"] += wall
            return
        for i, k in enumerate(PHASES):
            self.phase_seconds[k] += wall * float(d[i]) / tot

    def _step_host(self, actions, autoreset: bool) -> StepOutput:
        t0 = time.perf_counter()
        a = np.ascontiguousarray(actions, dtype=np.float64)
        want = (self.W, self.M, 3)
        if a.shape != want:
            raise ValueError(f"actions shape {a.shape}, expected {want}")
        bufs = self._host_bufs
        key = (bool(autoreset), self._metrics_on)
        io = self._host_io.get(key)
        if io is None:
            # the host path always uses the same device buffers: build its DgStepIO once
            # the host path's obs buffer is the engine's own: resident (zeroed at
            # construction, written only by these steps)
            io = self._host_io[key] = self._step_io(self._act_dev, bufs, autoreset=autoreset,
                                                    prefix_out=self._prefix_dev, resident=True,
                                                    phase_cycles=self._phase_dev)
        stream = torch.cuda.current_stream(self.device)
        slab = self._mapped_pool.acquire()
        t1 = time.perf_counter()
        # one host call: finiteness check while staging the actions in pinned memory
        # (raises before anything is queued, engine.py:291-294), H2D, the step and --
        # with a mapped slab -- the delivery: obs rows written into the slab by the
        # device (non-zero prefixes only), the packed per-tick outputs DMA'd behind them
        bad = ct.c_int64(-1)
        if slab is not None:
            ptr, prev, hb = slab
            ob = self._host_obs_bytes
            rc = self._lib.dg_step_host(self._h, ct.byref(io), a.ctypes.data, self._act_host.data_ptr(),
                                        ct.c_void_p(ptr), _ptr(prev), _ptr(self._host_bufs.aux),
                                        ct.c_void_p(ptr + ob), self._host_blob.numel() - ob, _ptr(self.d2h_bytes),
                                        ct.byref(bad), ct.c_void_p(stream.cuda_stream))
        else:
            rc = self._lib.dg_step_host(self._h, ct.byref(io), a.ctypes.data, self._act_host.data_ptr(),
                                        None, None, None, None, 0, None, ct.byref(bad),
                                        ct.c_void_p(stream.cuda_stream))
        if rc == N.DG_ENONFINITE and bad.value >= 0:
            w, m = divmod(bad.value // 3, self.M)
            raise ValueError(f"non-finite action for world {w} agent {m}")
        N.check(self._lib, rc, "dg_step_host")
        self._step_count += 1
        self.launches += 2 if slab is not None else 1
        if slab is None:
            host, hb = self._host_pool.acquire()
            host.copy_(self._host_blob, non_blocking=True)          # obs + every per-tick output, one copy
        stream.synchronize()
        t2 = time.perf_counter()
        obs = hb[:self.W * self.M * self.obs_config.obs_dim * 4].view(np.float32).reshape(bufs.obs.shape)
        hv = self._host_views(hb[self._host_obs_bytes:])
        src = hv
        src["step"] = self._step_count
        self.phase_seconds["action"] += t1 - t0
        self._phase_host = hb[self._phase_off:self._phase_off + 40].view(np.int64).copy()   # no view: the slab recycles
        self._book_phases(t2 - t1)
        return StepOutput(obs, hv["rewards"], hv["dones"].astype(bool), hv["events"], src, to_host=True)

    # ------------------------------------------------------------------ resets
    def teleport_reset(self, mask, new_starts=None, new_goals=None, new_headings=None):
        """Masked teleport reset (engine.py:599-619)."""
        dev = self.device

        def to_dev(a, dtype):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=dtype).contiguous()
            return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)

        m = to_dev(np.asarray(mask, dtype=bool) if not isinstance(mask, torch.Tensor) else mask, torch.uint8)
        N.check(self._lib, self._lib.dg_reset(self._h, _ptr(m), _ptr(to_dev(new_starts, torch.float64)),
                                              _ptr(to_dev(new_goals, torch.float64)),
                                              _ptr(to_dev(new_headings, torch.float64)), self._stream()),
                "dg_reset")
        self.launches += 1

    # ------------------------------------------------------------------ policies / episodes
    def lane_follower(self, obs: torch.Tensor, out: torch.Tensor | None = None, steer_gain=2.0,
                      throttle=0.5) -> torch.Tensor:
        """Device LaneFollower: float64 actions identical to the numpy policy."""
        acts = out if out is not None else torch.empty((self.W, self.M, 3), dtype=torch.float64,
                                                       device=self.device)
        N.check(self._lib, self._lib.dg_lane_follower(self._h, _ptr(obs), _ptr(acts), float(steer_gain),
                                                      float(throttle), self._stream()),
                "dg_lane_follower")
        self.launches += 1
        return acts

    # ------------------------------------------------------------------ episode metrics
    def track_episode_metrics(self, enable: bool = True) -> None:
        """Accumulate the episode safety metrics inside the step kernel: per
        agent, the running max of the pairwise DRAC of every tick's
        post-physics state over the agents alive before the tick, and goal /
        collision event latches (what episode_metrics derives from a recorded
        log, metrics.py:86-125).  Zeroes the accumulators."""
        self._metrics_on = bool(enable)
        self._host_io.clear()            # cached DgStepIO hold the accumulator pointers
        if enable:
            W, M = self.W, self.M
            self._drac_max = torch.zeros((W, M), dtype=torch.float64, device=self.device)
            self._metric_seen = torch.zeros((W, M), dtype=torch.uint8, device=self.device)

    def reset_episode_metrics(self) -> None:
        if self._metrics_on:
            self._drac_max.zero_()
            self._metric_seen.zero_()

    def episode_metrics(self, threshold: float = 3.4):
        """SR / CR / mean peak DRAC from the in-kernel accumulators
        (metrics.EpisodeMetrics, the reference's episode_metrics result)."""
        from .metrics import aggregate
        if not self._metrics_on:
            raise RuntimeError("episode metrics are not tracked: call track_episode_metrics() first")
        seen = self._metric_seen.cpu().numpy()
        return aggregate(seen & 1 != 0, seen & 2 != 0, self._drac_max.cpu().numpy(), self.valid, threshold)

    def run_episode(self, policy, record: bool = False, max_steps: int | None = None) -> "EpisodeLog":
        """Step until every agent terminated or the episode times out
        (engine.py:621-643); the log holds the per-step records when ``record``."""
        log = EpisodeLog(control_dt=self.config.control_dt)
        log.initial_state = {k: v.copy() for k, v in self.state.items() if k in LOG_STATE_FIELDS}
        limit = max_steps if max_steps is not None else self.config.episode_len
        obs = self.observe()
        for _ in range(limit):
            actions = policy(obs)
            out = self.step(actions)
            if record:
                log.append(self._step_count, out.info["state"], actions, out.rewards,
                           out.info["reward_terms"], out.events, out.dones, out.info["alive"],
                           out.info["alive_pre"])
            obs = out.obs
            if not out.info["alive"].any() or self._step_count >= self.config.episode_len:
                break
        return log


LOG_STATE_FIELDS = ("x", "y", "yaw", "v_x", "v_y", "yaw_rate", "steer_angle", "wheel_front", "wheel_rear")


class EpisodeLog:
    """Control-rate record of an episode (engine.py:83-145): per-step state
    snapshots taken before the teleport write-back, actions, rewards, terms,
    events, dones and alive masks."""

    def __init__(self, control_dt: float, initial_state: dict | None = None):
        self.control_dt = control_dt
        self.initial_state = initial_state
        self.steps = []

    def append(self, step, state, actions, rewards, terms, events, dones, alive, alive_pre):
        self.steps.append({
            "step": step,
            "state": {k: np.array(state[k]) for k in LOG_STATE_FIELDS},
            "actions": np.array(actions, dtype=np.float64),
            "rewards": np.array(rewards),
            "terms": {k: np.array(v) for k, v in terms.items()},
            "events": {k: np.array(v) for k, v in events.items()},
            "dones": np.array(dones),
            "alive": np.array(alive),
            "alive_pre": np.array(alive_pre),
        })

    def __len__(self):
        return len(self.steps)

    def resample_60hz(self) -> list:
        """States at twice the control rate by midpoint interpolation (engine.py:111-121)."""
        out, prev = [], self.initial_state
        for rec in self.steps:
            cur = rec["state"]
            if prev is not None:
                out.append({k: 0.5 * (prev[k] + cur[k]) for k in LOG_STATE_FIELDS})
            out.append({k: cur[k].copy() for k in LOG_STATE_FIELDS})
            prev = cur
        return out

    def to_jsonl(self, path):
        """One JSON record per (step, world, agent), full float precision (engine.py:123-145)."""
        import json
        with open(path, "w", encoding="utf-8") as fh:
            for rec in self.steps:
                W, M = rec["alive"].shape
                st = rec["state"]
                for w in range(W):
                    for m in range(M):
                        fh.write(json.dumps({
                            "step": rec["step"], "world": w, "agent": m,
                            "pose": [float(st["x"][w, m]), float(st["y"][w, m]), float(st["yaw"][w, m])],
                            "vel": [float(st["v_x"][w, m]), float(st["v_y"][w, m]),
                                    float(st["yaw_rate"][w, m])],
                            "action": rec["actions"][w, m].tolist(),
                            "reward": float(rec["rewards"][w, m]),
                            "terms": {k: float(v[w, m]) for k, v in rec["terms"].items()},
                            "events": [k for k, v in rec["events"].items() if v[w, m]],
                            "alive": bool(rec["alive"][w, m]),
                        }) + "\n")
