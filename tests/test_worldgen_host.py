"""The host restatement of world construction -- the checker of the on-device
build -- pinned to the reference's build_engine: every init
table at 4096x16 by sha256 (golden worlds_4096) and the scene_cases pool at 29
worlds in full (golden worlds_cases), with and without eval.random_goals.
Also the flattened pool the device build consumes."""

from __future__ import annotations

import numpy as np
import pytest

from cases import GOLDEN, canon, check_world_hashes, host_world_arrays, world_cfg, worlds_case_pool


@pytest.mark.parametrize("tag,goals", [("plain", None), ("goals", (15.0, 60.0))])
def test_host_build_4096_matches_reference(tag, goals):
    check_world_hashes(host_world_arrays(world_cfg(4096, goals=goals)), np.load(GOLDEN / "worlds_4096.npz"), tag)


@pytest.mark.parametrize("tag,goals", [("plain", None), ("goals", (10.0, 50.0))])
def test_host_build_scene_cases_match_reference(tag, goals):
    g = np.load(GOLDEN / "worlds_cases.npz")
    got = host_world_arrays(world_cfg(29, seed=7, goals=goals), worlds_case_pool())
    for k, v in got.items():
        assert np.array_equal(canon(v), g[f"{tag}__{k}"]), k


def test_flatten_pool_layout():
    from paper_2605_08528_b200.worldgen import flatten_pool, scene_order
    pool = worlds_case_pool()
    f = flatten_pool(pool)
    assert f["scene_poly"][-1] == len(f["poly_type"]) == sum(len(s.polylines) for s in pool)
    assert f["poly_start"][-1] == len(f["points"])
    assert f["scene_agent"][-1] == len(f["agents"]) == sum(len(s.agents) for s in pool)
    s1 = pool[1]
    a, b = f["poly_start"][f["scene_poly"][1]], f["poly_start"][f["scene_poly"][1] + 1]
    assert np.array_equal(f["points"][a:b], np.asarray(s1.polylines[0].points)[:, :2])
    from paper_2605_08528_b200.scenes import assign_scenes
    order = scene_order(len(pool), "random_fill", 7)
    assert np.array_equal(order[np.arange(29) % len(pool)], assign_scenes(29, len(pool), "random_fill", 7))
