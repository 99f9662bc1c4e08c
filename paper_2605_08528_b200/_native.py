"""ctypes binding of ``libdrivegrid_b200.so`` (C ABI: ``include/drivegrid_b200.h``).

This is the binding a maintainer of the reference would add: plain ctypes
over the extern "C" entry points, no torch types in any signature.  The
library is built in-tree by ``build_native()`` (nvcc, sm_100a); a missing or
stale library is a hard error -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as ct
import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_PATH = PKG / "libdrivegrid_b200.so"
SOURCES = [PKG / "csrc" / "drivegrid_b200.cu", PKG / "csrc" / "dg_policy.cu", PKG / "csrc" / "dg_worlds.cu"]
DEPS = [PKG / "csrc" / "dg_fastmath.cuh", PKG / "csrc" / "dg_umma.cuh"]
HEADER = ROOT / "include" / "drivegrid_b200.h"
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-fmad=false", "-Xcompiler", "-fPIC", "-shared"]

DG_OK, DG_EINVAL, DG_ENONFINITE, DG_ECUDA, DG_ENOSUPPORT = 0, 1, 2, 3, 4
DG_NO_ERROR = 0x7FFFFFFF
ABI_VERSION = 13


class DgDims(ct.Structure):
    _fields_ = [(n, ct.c_int32) for n in (
        "W", "M", "obs_dim", "ego_dim", "k_road", "k_vehicles", "include_weather", "dynamic",
        "decimation", "episode_len", "invincible", "collision_warmup", "num_scenes",
        "max_scene_bytes", "max_segments", "geometry_global")]


CONST_FIELDS = (
    "physics_dt", "control_dt",
    "kp_steer", "kd_steer", "theta_max", "tau_steer_max", "steer_inertia", "steer_limit",
    "a_f", "b_r", "tau_drive_max", "tau_brake_front", "tau_brake_rear", "wheel_radius",
    "cornering_stiffness", "f_z", "chassis_mass", "lambda_lat", "lambda_yaw", "yaw_inertia",
    "i_axle", "wheelbase",
    "bic_a_max", "bic_b_max", "bic_c_roll", "bic_steer_max",
    "road_radius", "road_radius_sq", "bbox_half", "speed_norm", "type_norm", "ttc_max",
    "goal_radius", "goal_weight", "collision_weight", "crash_weight", "crash_drift_limit",
    "lane_forbidden_weight", "progress_weight", "progress_clamp", "lane_weight", "lane_sigma",
    "lane_heading_weight", "lane_heading_base", "offroad_weight", "offroad_lat_limit",
    "offroad_dist_limit", "idle_weight", "idle_speed", "ttc_vehicle_alpha", "ttc_vehicle_pmax",
    "ttc_edge_alpha", "ttc_edge_pmax", "ttc_floor", "edge_range", "crash_speed_limit", "offstage_x",
)


class DgConsts(ct.Structure):
    _fields_ = [(n, ct.c_double) for n in CONST_FIELDS]


_P = ct.c_void_p


class DgEngineDesc(ct.Structure):
    _fields_ = [("dims", DgDims), ("k", DgConsts)] + [(n, _P) for n in (
        "scene_blob", "scene_meta", "scene_of_world", "grid_offset", "mu_eff", "weather", "valid",
        "length", "width", "r_hull", "d_hull", "state", "alive", "reason", "event_seen",
        "spawn_step", "step_count", "start_xy", "goal_xy", "start_yaw", "error_word", "scratch")]


POL_SECTIONS = ("W_EGO1", "W_EGO2", "W_T1", "W_T2", "W_ROAD1", "W_ROAD2", "W_VEH1", "W_VEH2",
                "B_EGO1", "B_EGO2", "B_ROAD1", "B_ROAD2", "B_VEH1", "B_VEH2", "B_T1", "B_T2",
                "W_HEAD", "B_HEAD", "LOG_STD")


class DgPolicyDesc(ct.Structure):
    _fields_ = [(n, ct.c_int32) for n in ("n_agents", "obs_dim", "ego_dim", "k_road", "k_vehicles", "critic")] + [
        ("obs", _P), ("weights", _P), ("net_stride", ct.c_int64), ("off", ct.c_int64 * len(POL_SECTIONS)),
        ("emb", _P), ("mean", _P), ("actions", _P), ("value", _P),
        ("sample", ct.c_int32), ("first_net", ct.c_int32), ("seed", ct.c_uint64), ("counter", ct.c_uint64),
        ("log_prob", _P), ("actions_f32", _P), ("prefix", _P), ("work_counter", _P)]


class DgStepIO(ct.Structure):
    _fields_ = [("actions", _P), ("actions_f64", ct.c_int32), ("autoreset", ct.c_int32)] + [
        (n, _P) for n in ("obs", "rewards", "dones", "events", "reason_out", "alive_out",
                          "alive_pre_out", "ttc_min_out", "terms_out", "snapshot_out",
                          "next_actions")] + [("policy_gain", ct.c_double), ("policy_throttle", ct.c_double),
                                              ("event_counts", _P),
                                              ("ticks", ct.c_int32), ("ring_slots", ct.c_int32),
                                              ("ring_start", ct.c_int32), ("obs_resident", ct.c_int32),
                                              ("drac_max", _P), ("metric_seen", _P), ("index_out", _P),
                                              ("prefix_out", _P), ("phase_cycles", _P)]


class DgScenePool(ct.Structure):
    _fields_ = [(n, ct.c_int32) for n in ("num_scenes", "num_polylines", "num_points", "num_agents")] + [
        (n, _P) for n in ("points", "poly_start", "poly_type", "scene_poly", "agents", "scene_agent")]


class DgSceneBuild(ct.Structure):
    _fields_ = [(n, ct.c_double) for n in ("gap", "bbox_half", "half_width", "goal_radius")] + [
        ("cap", ct.c_int32), ("pad_", ct.c_int32)]


SCENE_SEG_FIELDS = ("mid", "dir", "type", "half_len", "half_wid", "lane_index", "edge_index", "arc",
                    "seg_count", "lane_count", "edge_count", "lane_polys", "kept_count", "kept_agent")


class DgSceneSegments(ct.Structure):
    _fields_ = [(n, _P) for n in SCENE_SEG_FIELDS]


WORLD_OUT_FIELDS = ("assignment", "grid_offset", "valid", "alive", "start_xy", "goal_xy", "start_yaw",
                    "length", "width", "r_hull", "d_hull", "state")
WORLD_OPT_FIELDS = ("wb_mid", "wb_dir", "wb_type", "wb_half_len", "wb_half_wid", "wb_mask",
                    "lane_mid", "lane_dir", "lane_half_len", "lane_half_wid", "lane_mask",
                    "edge_mid", "edge_dir", "edge_half_len", "edge_half_wid", "edge_mask")


class DgWorldBuild(ct.Structure):
    _fields_ = ([(n, ct.c_int32) for n in ("W", "M", "num_scenes", "grid_cols")] + [("world_base", ct.c_int64)]
                + [(n, ct.c_double) for n in ("pitch", "offstage_x", "wheelbase")] + [("scene_order", _P)]
                + [(n, _P) for n in WORLD_OUT_FIELDS]
                + [("random_goals", ct.c_int32), ("pad_", ct.c_int32), ("goal_min", ct.c_double),
                   ("goal_max", ct.c_double), ("goal_draws", _P)]
                + [(n, ct.c_int32) for n in ("p_max", "k_lane", "k_edge", "pad2_")]
                + [(n, _P) for n in WORLD_OPT_FIELDS])


# exported symbol -> (restype, argtypes)
SIGNATURES = {
    "dg_abi_version": (ct.c_int, []),
    "dg_last_error": (ct.c_char_p, []),
    "dg_create": (ct.c_int, [ct.POINTER(DgEngineDesc), ct.POINTER(_P)]),
    "dg_destroy": (ct.c_int, [_P]),
    "dg_step": (ct.c_int, [_P, ct.POINTER(DgStepIO), _P]),
    "dg_observe": (ct.c_int, [_P, _P, _P, _P, ct.c_double, ct.c_double, _P]),
    "dg_reset": (ct.c_int, [_P, _P, _P, _P, _P, _P]),
    "dg_get_state": (ct.c_int, [_P, _P, _P]),
    "dg_set_state": (ct.c_int, [_P, _P, _P]),
    "dg_set_step_count": (ct.c_int, [_P, ct.c_int32, _P]),
    "dg_check_actions": (ct.c_int, [_P, _P, ct.c_int32, _P]),
    "dg_read_error": (ct.c_int, [_P, ct.POINTER(ct.c_int32), _P]),
    "dg_lane_follower": (ct.c_int, [_P, _P, _P, ct.c_double, ct.c_double, _P]),
    "dg_launch_count": (ct.c_int, [_P]),
    "dg_tune": (ct.c_int, [_P, ct.c_int32, ct.c_int32, ct.c_int32]),
    "dg_scratch_bytes": (ct.c_size_t, [ct.c_int32, ct.c_int32]),
    "dg_index_stride": (ct.c_int32, [_P]),
    "dg_sysid_rollout": (ct.c_int, [_P] * 6 + [ct.c_int32, ct.c_int32, _P, _P]),
    "dg_policy_forward": (ct.c_int, [ct.POINTER(DgPolicyDesc), _P]),
    "dg_policy_scratch_bytes": (ct.c_size_t, [ct.c_int32, ct.c_int32]),
    "dg_policy_last_error": (ct.c_char_p, []),
    "dg_gae": (ct.c_int, [_P, _P, _P, ct.c_int32, ct.c_int64, ct.c_double, ct.c_double, _P, _P, _P]),
    "dg_pairwise_drac": (ct.c_int, [_P] * 8 + [ct.c_int32, ct.c_int32, ct.c_int32, _P, ct.c_int32, ct.c_int32, _P]),
    "dg_host_alloc": (ct.c_int, [ct.c_size_t, ct.POINTER(_P)]),
    "dg_host_free": (ct.c_int, [_P]),
    "dg_to_host": (ct.c_int, [_P, _P, _P, _P, _P, _P, _P, ct.c_size_t, _P, _P]),
    "dg_step_host": (ct.c_int, [_P, ct.POINTER(DgStepIO), _P, _P, _P, _P, _P, _P, ct.c_size_t, _P,
                                ct.POINTER(ct.c_int64), _P]),
    "dg_lane_follower_rows": (ct.c_int, [_P, ct.c_int64, ct.c_int32, ct.c_double, ct.c_double, ct.c_double, _P]),
    "dg_build_scenes": (ct.c_int, [ct.POINTER(DgScenePool), ct.POINTER(DgSceneBuild), ct.POINTER(DgSceneSegments),
                                   _P]),
    "dg_build_worlds": (ct.c_int, [ct.POINTER(DgScenePool), ct.POINTER(DgSceneSegments), ct.POINTER(DgWorldBuild),
                                   _P]),
}


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + DEPS + [HEADER] if p.exists())


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile the CUDA library in-tree for sm_100a (works without a GPU)."""
    if not force and not _stale():
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-o", str(LIB_PATH) + ".tmp",
           *map(str, SOURCES)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{proc.stderr}")
    os.replace(str(LIB_PATH) + ".tmp", LIB_PATH)
    if verbose:
        print(proc.stderr)
    return LIB_PATH


_LIB = None


def load_library(build_if_missing: bool = True) -> ct.CDLL:
    """The native library; raises if it cannot be built or loaded."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if build_if_missing and _stale():
        build_native()
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} missing: run paper_2605_08528_b200._native.build_native()")
    lib = ct.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.dg_abi_version() != ABI_VERSION:
        raise RuntimeError("libdrivegrid_b200.so ABI version mismatch; rebuild it")
    _LIB = lib
    return lib


class NativeError(RuntimeError):
    pass


def check(lib, status: int, what: str) -> None:
    if status == DG_OK:
        return
    msg = (lib.dg_last_error() or b"").decode()
    if status == DG_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed (status {status}): {msg}")
