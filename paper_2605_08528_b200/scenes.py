"""Scenario records, procedural scenes and the world-batch builder (host, init only).

This is the input producer of the hot path: it turns typed road polylines
into oriented segments and lays W worlds out on the 400 m grid.  It runs once
per engine, on the host, in float64 numpy, with the same operation order as
the reference so the geometry handed to the GPU is bit-identical to the
geometry the reference engine steps against.

Reference anchors (``/root/reference/pkg/src/drivegrid``):
  * schema / filters      scenario.py:29-101, 152-192, 208-271
  * procedural scenes     synth.py:10-90
  * world build           world.py:59-194 (recenter, flatten_z, segmentize,
                          grid_offsets, assign_scenes, build_world_batch)
  * binary export         world.py:199-236
"""

from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .params import LANE_CENTER_CODES

SEGMENT_GAP = 3.0
SEGMENT_HALF_WIDTH = 0.05
GRID_PITCH = 400.0
EXPORT_VERSION = 1
DEFAULT_AGENT_LENGTH = 4.0
DEFAULT_AGENT_WIDTH = 2.0


class ScenarioError(ValueError):
    """A scenario file failed schema validation."""


# ----------------------------------------------------------------------------
# schema
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class Polyline:
    type_code: int
    points: np.ndarray  # (N, 3) float64

    def __post_init__(self):
        pts = np.asarray(self.points, dtype=np.float64)
        object.__setattr__(self, "points", pts)
        if pts.ndim != 2 or pts.shape[1] != 3 or pts.shape[0] < 2:
            raise ScenarioError(f"polyline needs >=2 points of (x, y, z); got shape {pts.shape}")
        if not np.isfinite(pts).all():
            raise ScenarioError("polyline contains non-finite coordinates")


@dataclass(frozen=True)
class AgentRecord:
    id: str
    start: tuple
    start_heading: float
    goal: tuple
    length: float = DEFAULT_AGENT_LENGTH
    width: float = DEFAULT_AGENT_WIDTH

    def __post_init__(self):
        vals = (*self.start, self.start_heading, *self.goal, self.length, self.width)
        if not all(math.isfinite(v) for v in vals):
            raise ScenarioError(f"agent {self.id!r} has non-finite fields")
        if self.length <= 0 or self.width <= 0:
            raise ScenarioError(f"agent {self.id!r} has non-positive dimensions")


@dataclass(frozen=True)
class ScenarioSpec:
    scenario_id: str
    polylines: list
    agents: list = field(default_factory=list)

    def __post_init__(self):
        if not self.scenario_id:
            raise ScenarioError("scenario_id must be non-empty")
        if not self.polylines:
            raise ScenarioError("scenario has no polylines")

    def lane_polylines(self) -> list:
        return [p for p in self.polylines if p.type_code in LANE_CENTER_CODES]

    def to_dict(self) -> dict:
        return {
            "scenario_id": self.scenario_id,
            "polylines": [{"type": int(p.type_code), "points": p.points.tolist()}
                          for p in self.polylines],
            "agents": [{"id": a.id, "start": list(a.start), "start_heading": a.start_heading,
                        "goal": list(a.goal), "length": a.length, "width": a.width}
                       for a in self.agents],
        }


def scenario_from_dict(raw: dict) -> ScenarioSpec:
    """Validated spec from parsed JSON (scenario.py:108-149)."""
    def need(cond, msg):
        if not cond:
            raise ScenarioError(msg)

    need(isinstance(raw, dict), "scenario root must be a JSON object")
    need("scenario_id" in raw, "missing field 'scenario_id'")
    need("polylines" in raw, "missing field 'polylines'")
    sid = raw["scenario_id"]
    need(isinstance(sid, str) and sid != "", "'scenario_id' must be a non-empty string")
    polys = []
    for i, entry in enumerate(raw["polylines"]):
        need(isinstance(entry, dict), f"polylines[{i}] must be an object")
        need("type" in entry, f"polylines[{i}] missing field 'type'")
        need("points" in entry, f"polylines[{i}] missing field 'points'")
        try:
            polys.append(Polyline(int(entry["type"]), np.asarray(entry["points"], dtype=np.float64)))
        except (TypeError, ValueError) as exc:
            raise ScenarioError(f"polylines[{i}]: {exc}") from exc
    agents = []
    for i, entry in enumerate(raw.get("agents", [])):
        need(isinstance(entry, dict), f"agents[{i}] must be an object")
        for key in ("id", "start", "start_heading", "goal"):
            need(key in entry, f"agents[{i}] missing field '{key}'")
        try:
            agents.append(AgentRecord(
                id=str(entry["id"]),
                start=(float(entry["start"][0]), float(entry["start"][1])),
                start_heading=float(entry["start_heading"]),
                goal=(float(entry["goal"][0]), float(entry["goal"][1])),
                length=float(entry.get("length", DEFAULT_AGENT_LENGTH)),
                width=float(entry.get("width", DEFAULT_AGENT_WIDTH))))
        except (TypeError, ValueError, IndexError) as exc:
            raise ScenarioError(f"agents[{i}]: {exc}") from exc
    return ScenarioSpec(sid, polys, agents)


def load_scenario(path) -> ScenarioSpec:
    path = Path(path)
    try:
        raw = json.loads(path.read_text(encoding="utf-8"))
    except json.JSONDecodeError as exc:
        raise ScenarioError(f"{path}: not valid JSON ({exc})") from exc
    try:
        return scenario_from_dict(raw)
    except ScenarioError as exc:
        raise ScenarioError(f"{path}: {exc}") from exc


def save_scenario(spec: ScenarioSpec, path) -> None:
    Path(path).write_text(json.dumps(spec.to_dict()), encoding="utf-8")


def filter_agents(spec: ScenarioSpec, bbox_half=100.0, goal_radius=3.0, cap=16) -> list:
    """Spawn filter: in-bounds endpoints, start-goal gap > goal_radius,
    file order, first ``cap`` (scenario.py:169-192)."""
    kept = []
    for a in spec.agents:
        if max(abs(a.start[0]), abs(a.start[1]), abs(a.goal[0]), abs(a.goal[1])) > bbox_half:
            continue
        if math.dist(a.start, a.goal) <= goal_radius:
            continue
        kept.append(a)
        if len(kept) == cap:
            break
    return kept


def shift_scenario(spec: ScenarioSpec, dx: float, dy: float) -> ScenarioSpec:
    polys = []
    for p in spec.polylines:
        pts = p.points.copy()
        pts[:, 0] += dx
        pts[:, 1] += dy
        polys.append(Polyline(p.type_code, pts))
    agents = [replace(a, start=(a.start[0] + dx, a.start[1] + dy),
                      goal=(a.goal[0] + dx, a.goal[1] + dy)) for a in spec.agents]
    return ScenarioSpec(spec.scenario_id, polys, agents)


def recenter(spec: ScenarioSpec):
    """Shift so the mean polyline point is the origin (world.py:59-68)."""
    pts = np.concatenate([p.points[:, :2] for p in spec.polylines], axis=0)
    if pts.size == 0:
        raise ValueError("scenario has no polyline points")
    cx, cy = pts.mean(axis=0)
    return shift_scenario(spec, -cx, -cy), (float(cx), float(cy))


def flatten_z(spec: ScenarioSpec):
    zs = [p.points[:, 2].copy() for p in spec.polylines]
    flat = []
    for p in spec.polylines:
        pts = p.points.copy()
        pts[:, 2] = 0.0
        flat.append(Polyline(p.type_code, pts))
    return ScenarioSpec(spec.scenario_id, flat, spec.agents), zs


@dataclass(frozen=True)
class SceneVerdict:
    accepted: bool
    reason: str = ""


def reject_degenerate_scene(spec: ScenarioSpec, bbox_half=100.0, goal_radius=3.0, cap=16,
                            z_gap=3.0, overlap_fraction=0.20, overlap_radius=1.0) -> SceneVerdict:
    """No lanes / multi-level proxy / no spawnable agent (scenario.py:208-252)."""
    if not spec.lane_polylines():
        return SceneVerdict(False, "no drivable lanes")
    mids = []
    for p in spec.polylines:
        m = 0.5 * (p.points[:-1] + p.points[1:])
        mids.append((m[:, :2], m[:, 2]))
    coincident = 0
    stacked = 0
    for i in range(len(mids)):
        for j in range(i + 1, len(mids)):
            d2 = ((mids[i][0][:, None, :] - mids[j][0][None, :, :]) ** 2).sum(axis=2)
            close = d2 < overlap_radius ** 2
            if not close.any():
                continue
            dz = np.abs(mids[i][1][:, None] - mids[j][1][None, :])
            coincident += int(close.sum())
            stacked += int((close & (dz > z_gap)).sum())
    if coincident > 0 and stacked / coincident > overlap_fraction:
        return SceneVerdict(False, f"multi-level overlap ({stacked}/{coincident} coincident pairs z-separated)")
    centered, _ = recenter(spec)
    if not filter_agents(centered, bbox_half=bbox_half, goal_radius=goal_radius, cap=cap):
        return SceneVerdict(False, "no valid agents after spawn filter")
    return SceneVerdict(True)


def prepare_scene(spec: ScenarioSpec):
    """Degeneracy filter, recenter, flatten (config.py:162-168); None if rejected."""
    if not reject_degenerate_scene(spec).accepted:
        return None
    centered, _ = recenter(spec)
    flat, _ = flatten_z(centered)
    return flat


# ----------------------------------------------------------------------------
# procedural scenes (synth.py:10-90)
# ----------------------------------------------------------------------------

def _row(xs, y):
    return np.stack([xs, np.full_like(xs, y), np.zeros_like(xs)], axis=1)


def straight_scene(scenario_id="straight", half_length=80.0, lane_spacing=2.0,
                   lane_offsets=(0.0,), edge_offset=6.0, agent_count=1,
                   agent_gap=12.0, goal_dist=50.0) -> ScenarioSpec:
    """East-west road: lane centres (code 1) plus two edges (code 15)."""
    xs = np.arange(-half_length, half_length + 1e-9, lane_spacing)
    polys = [Polyline(1, _row(xs, off)) for off in lane_offsets]
    polys += [Polyline(15, _row(xs, sgn * edge_offset)) for sgn in (1.0, -1.0)]
    agents = []
    for i in range(agent_count):
        lane = lane_offsets[i % len(lane_offsets)]
        x0 = -half_length + 10.0 + i * agent_gap
        agents.append(AgentRecord(f"a{i}", (x0, lane), 0.0, (x0 + goal_dist, lane)))
    return ScenarioSpec(scenario_id, polys, agents)


def crossroads_scene(scenario_id="crossroads", half_length=80.0, agent_count=4,
                     goal_dist=40.0) -> ScenarioSpec:
    """Two perpendicular lanes through the origin, agents alternating arms."""
    xs = np.arange(-half_length, half_length + 1e-9, 2.0)
    zero = np.zeros_like(xs)
    ew = Polyline(1, np.stack([xs, zero, zero], axis=1))
    ns = Polyline(2, np.stack([zero, xs, zero], axis=1))
    edges = [Polyline(15, _row(xs, off)) for off in (half_length * 0.9, -half_length * 0.9)]
    agents = []
    for i in range(agent_count):
        s = -half_length + 15.0 + (i // 2) * 9.0
        if i % 2 == 0:
            agents.append(AgentRecord(f"a{i}", (s, 0.0), 0.0, (s + goal_dist, 0.0)))
        else:
            agents.append(AgentRecord(f"a{i}", (0.0, s), np.pi / 2, (0.0, s + goal_dist)))
    return ScenarioSpec(scenario_id, [ew, ns, *edges], agents)


def two_level_scene(scenario_id="overpass", dz=6.0) -> ScenarioSpec:
    xs = np.arange(-40.0, 40.0 + 1e-9, 2.0)
    low = Polyline(1, np.stack([xs, np.zeros_like(xs), np.zeros_like(xs)], axis=1))
    high = Polyline(2, np.stack([xs, np.zeros_like(xs), np.full_like(xs, dz)], axis=1))
    return ScenarioSpec(scenario_id, [low, high], [AgentRecord("a0", (-30.0, 0.0), 0.0, (20.0, 0.0))])


def default_scene_pool(n=4, agent_count=16) -> list:
    """Built-in pool: straight / crossroads alternating (synth.py:81-90)."""
    pool = []
    for i in range(n):
        if i % 2 == 0:
            pool.append(straight_scene(f"synth-straight-{i}", agent_count=agent_count,
                                       agent_gap=8.0, lane_offsets=(0.0, 4.0, -4.0)))
        else:
            pool.append(crossroads_scene(f"synth-cross-{i}", agent_count=agent_count))
    return pool


# ----------------------------------------------------------------------------
# segments and the world grid
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class SegmentArray:
    midpoints: np.ndarray
    directions: np.ndarray
    type_codes: np.ndarray
    half_lengths: np.ndarray
    half_widths: np.ndarray

    def __len__(self):
        return self.midpoints.shape[0]


def segmentize(polyline: Polyline, gap=SEGMENT_GAP, bbox_half=100.0) -> SegmentArray:
    """Consecutive point pairs -> oriented boxes; long or out-of-box pairs dropped
    (world.py:82-109)."""
    pts = polyline.points[:, :2]
    a, b = pts[:-1], pts[1:]
    diff = b - a
    length = np.sqrt((diff ** 2).sum(axis=1))
    inside = (np.abs(a) <= bbox_half).all(axis=1) & (np.abs(b) <= bbox_half).all(axis=1)
    keep = (length > 0.0) & (length <= gap) & inside
    a, b, diff, length = a[keep], b[keep], diff[keep], length[keep]
    n = len(length)
    return SegmentArray(0.5 * (a + b), diff / length[:, None],
                        np.full(n, polyline.type_code, dtype=np.int32),
                        0.5 * length, np.full(n, SEGMENT_HALF_WIDTH))


def scene_segments(spec: ScenarioSpec, gap=SEGMENT_GAP, bbox_half=100.0) -> SegmentArray:
    parts = [segmentize(p, gap=gap, bbox_half=bbox_half) for p in spec.polylines]
    if not parts:
        return SegmentArray(np.zeros((0, 2)), np.zeros((0, 2)), np.zeros(0, np.int32),
                            np.zeros(0), np.zeros(0))
    return SegmentArray(*(np.concatenate([getattr(s, f) for s in parts])
                          for f in ("midpoints", "directions", "type_codes",
                                    "half_lengths", "half_widths")))


def grid_offsets(num_worlds: int, pitch=GRID_PITCH) -> np.ndarray:
    cols = int(np.ceil(np.sqrt(num_worlds)))
    idx = np.arange(num_worlds)
    return np.stack([(idx % cols) * pitch, (idx // cols) * pitch], axis=1).astype(np.float64)


def assign_scenes(num_worlds: int, num_scenes: int, mode: str, seed=42) -> np.ndarray:
    """World -> scene map; ``random_fill`` permutes the pool on Philox stream
    (seed, 0) (world.py:131-145)."""
    if num_scenes == 0:
        raise ValueError("empty scene list")
    if mode == "fixed":
        return np.arange(num_worlds) % num_scenes
    if mode == "random_fill":
        gen = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, 0])))
        return gen.permutation(num_scenes)[np.arange(num_worlds) % num_scenes]
    raise ValueError(f"unknown assignment mode {mode!r}")


@dataclass(frozen=True)
class WorldBatch:
    """Padded (W, P_max) geometry in scene-local coordinates + grid offsets.

    ``scene_tables`` keeps the un-padded per-scene segment arrays: worlds that
    share a scene share one device copy (the GPU never sees the padded form).
    """

    midpoints: np.ndarray
    directions: np.ndarray
    type_codes: np.ndarray
    half_lengths: np.ndarray
    half_widths: np.ndarray
    mask: np.ndarray
    grid_offsets: np.ndarray
    scenario_ids: list
    scene_index: np.ndarray | None = None      # (W,) index into scene_tables
    scene_tables: tuple | None = None           # per-scene SegmentArray

    @property
    def num_worlds(self) -> int:
        return self.midpoints.shape[0]

    @property
    def p_max(self) -> int:
        return self.midpoints.shape[1]


def build_world_batch(scenes, num_worlds, mode="random_fill", seed=42, gap=SEGMENT_GAP,
                      bbox_half=100.0):
    """Assemble W worlds from pre-centred scenes (world.py:148-194)."""
    assignment = assign_scenes(num_worlds, len(scenes), mode, seed)
    tables = [scene_segments(s, gap=gap, bbox_half=bbox_half) for s in scenes]
    used = sorted(set(assignment.tolist()))
    p_max = max(1, max(len(tables[i]) for i in used))
    W = num_worlds
    mid = np.zeros((W, p_max, 2))
    dirs = np.zeros((W, p_max, 2))
    codes = np.zeros((W, p_max), dtype=np.int32)
    hl = np.zeros((W, p_max))
    hw = np.zeros((W, p_max))
    mask = np.zeros((W, p_max), dtype=bool)
    for s_idx in used:
        seg = tables[s_idx]
        rows = np.nonzero(assignment == s_idx)[0]
        n = len(seg)
        mid[rows, :n] = seg.midpoints
        dirs[rows, :n] = seg.directions
        codes[rows, :n] = seg.type_codes
        hl[rows, :n] = seg.half_lengths
        hw[rows, :n] = seg.half_widths
        mask[rows, :n] = True
    ids = [scenes[i].scenario_id for i in assignment]
    batch = WorldBatch(mid, dirs, codes, hl, hw, mask, grid_offsets(W), ids,
                       scene_index=np.asarray(assignment, dtype=np.int64),
                       scene_tables=tuple(tables))
    return batch, assignment


def export_world_batch(batch: WorldBatch, path) -> None:
    """Little-endian header + f32/i32 arrays + packed mask (world.py:199-212)."""
    with open(path, "wb") as f:
        f.write(struct.pack("<III", batch.num_worlds, batch.p_max, EXPORT_VERSION))
        for arr, dt in ((batch.midpoints, "<f4"), (batch.directions, "<f4"),
                        (batch.type_codes, "<i4"), (batch.half_lengths, "<f4"),
                        (batch.half_widths, "<f4")):
            f.write(arr.astype(dt).tobytes())
        f.write(np.packbits(batch.mask.reshape(-1)).tobytes())
        f.write(batch.grid_offsets.astype("<f4").tobytes())


def import_world_batch(path) -> WorldBatch:
    data = Path(path).read_bytes()
    W, P, version = struct.unpack_from("<III", data, 0)
    if version != EXPORT_VERSION:
        raise ValueError(f"unsupported export version {version}")
    off = 12

    def take(count, dtype):
        nonlocal off
        arr = np.frombuffer(data, dtype=dtype, count=count, offset=off)
        off += arr.nbytes
        return arr

    mid = take(W * P * 2, "<f4").reshape(W, P, 2).astype(np.float64)
    dirs = take(W * P * 2, "<f4").reshape(W, P, 2).astype(np.float64)
    codes = take(W * P, "<i4").reshape(W, P).astype(np.int32)
    hl = take(W * P, "<f4").reshape(W, P).astype(np.float64)
    hw = take(W * P, "<f4").reshape(W, P).astype(np.float64)
    mask = np.unpackbits(take((W * P + 7) // 8, np.uint8), count=W * P).reshape(W, P).astype(bool)
    offs = take(W * 2, "<f4").reshape(W, 2).astype(np.float64)
    return WorldBatch(mid, dirs, codes, hl, hw, mask, offs, ["?"] * W)
