"""Scene intake on the host (no GPU): the degeneracy verdicts, recentring /
flattening and the spawn filter for synthetic specs covering every verdict
(lanes missing, multi-level overlap, goals out of the box, more than 16
agents, off-centre and elevated scenes), against the reference's own outputs
(tests/golden/scene_verdicts.npz, make_golden.py scene_verdicts)."""

from __future__ import annotations

import json
import sys
import types

import numpy as np

from cases import GOLDEN
from paper_2605_08528_b200 import scenes as S

sys.path.insert(0, str(GOLDEN))
from scene_cases import scene_specs  # noqa: E402


def test_scene_verdicts_and_prepared_scenes_match_reference():
    g = np.load(GOLDEN / "scene_verdicts.npz")
    want = json.loads(bytes(g["meta_json"]).decode())
    mod = types.SimpleNamespace(Polyline=S.Polyline, AgentRecord=S.AgentRecord, ScenarioSpec=S.ScenarioSpec,
                                straight_scene=S.straight_scene, crossroads_scene=S.crossroads_scene,
                                two_level_scene=S.two_level_scene, shift_scenario=S.shift_scenario)
    specs = scene_specs(mod)
    assert len(specs) == len(want)
    for i, (spec, w) in enumerate(zip(specs, want)):
        v = S.reject_degenerate_scene(spec)
        assert (spec.scenario_id, bool(v.accepted), v.reason) == (w["id"], w["accepted"], w["reason"])
        p = S.prepare_scene(spec)
        assert (p is not None) == w["accepted"]
        if p is None:
            continue
        assert len(S.filter_agents(p)) == w["kept"], w["id"]
        assert np.array_equal(np.concatenate([q.points for q in p.polylines]), g[f"s{i}_points"]), w["id"]
        agents = np.array([[*a.start, a.start_heading, *a.goal, a.length, a.width] for a in p.agents])
        assert np.array_equal(agents, g[f"s{i}_agents"]), w["id"]
