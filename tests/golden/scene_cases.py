"""Synthetic scene specs shared by make_golden.py (built with the reference's
classes) and tests/test_scene_host.py (built with this package's): the same
constructor calls on either module set give the same scenes."""

from __future__ import annotations

import numpy as np


def scene_specs(M) -> list:
    """``M``: a namespace with Polyline, AgentRecord, ScenarioSpec,
    straight_scene, crossroads_scene, two_level_scene, shift_scenario."""
    xs = np.arange(-60.0, 60.01, 2.0)

    def row(y, z=0.0):
        return np.stack([xs, np.full_like(xs, y), np.full_like(xs, z)], axis=1)

    specs = [
        M.straight_scene("plain", agent_count=3),
        M.crossroads_scene("cross", agent_count=6),
        M.two_level_scene("overpass", dz=6.0),
        M.two_level_scene("ramp", dz=2.0),
        M.ScenarioSpec("edges_only", [M.Polyline(15, row(5.0)), M.Polyline(16, row(-5.0))],
                       [M.AgentRecord("a0", (-40.0, 0.0), 0.0, (0.0, 0.0))]),
        M.ScenarioSpec("far_goals", [M.Polyline(1, row(0.0))],
                       [M.AgentRecord("a0", (-40.0, 0.0), 0.0, (400.0, 0.0))]),
        M.ScenarioSpec("crowd", [M.Polyline(1, row(0.0)), M.Polyline(2, row(4.0))],
                       [M.AgentRecord(f"a{i}", (-58.0 + 6.0 * i, 4.0 * (i % 2)), 0.0,
                                      (-38.0 + 6.0 * i, 4.0 * (i % 2))) for i in range(20)]),
        M.shift_scenario(M.straight_scene("shifted", agent_count=4, lane_offsets=(0.0, 3.5)), 350.0, -120.0),
        M.ScenarioSpec("hilly", [M.Polyline(1, row(0.0, 12.0)), M.Polyline(2, row(3.5, 12.5))],
                       [M.AgentRecord("a0", (-30.0, 0.0), 0.1, (10.0, 0.0), 4.5, 1.9)]),
    ]
    return specs
