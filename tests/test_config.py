"""Configuration surface mirrors the reference (engine.py:45-107,
observation.py:51-99, env.py:32-63)."""

import math

import pytest

from paper_2408_01584_b200.config import (EGO_WIDTH, PARTNER_WIDTH, RAY_WIDTH, ROAD_SLOT_WIDTH,
                                          ObsConfig, SimConfig, layout, obs_width)


def test_defaults_match_reference():
    c = SimConfig()
    assert (c.dynamics, c.goal_tolerance, c.collision_behavior, c.init_mode) == \
        ("classic", 2.0, "ignore", "all_nontrivial")
    assert c.accel_bounds == (-4.0, 4.0) and c.steer_bounds == (-0.7, 0.7) and c.v_max == 100.0
    o = ObsConfig()
    assert (o.mode, o.radius, o.n_rays, o.max_range, o.max_agents_obs, o.max_road_points_obs) == \
        ("radial", 50.0, 64, 100.0, 16, 64)
    assert o.fov == pytest.approx(2 * math.pi / 3)


@pytest.mark.parametrize("kw", [dict(dynamics="bogus"), dict(collision_behavior="x"),
                                dict(init_mode="y"), dict(goal_tolerance=0.0)])
def test_invalid_sim_config_raises(kw):
    with pytest.raises(ValueError):
        SimConfig(**kw)


@pytest.mark.parametrize("kw", [dict(mode="sonar"), dict(n_rays=0), dict(fov=0.0),
                                dict(fov=7.0)])
def test_invalid_obs_config_raises(kw):
    with pytest.raises(ValueError):
        ObsConfig(**kw)


def test_layout_widths():
    assert obs_width(ObsConfig()) == 823
    assert obs_width(ObsConfig(mode="lidar", n_rays=64)) == EGO_WIDTH + 64 * RAY_WIDTH == 327
    lay = layout(ObsConfig(max_agents_obs=4, max_road_points_obs=5))
    assert lay.offset("partners") == EGO_WIDTH
    assert lay.offset("roads") == EGO_WIDTH + 4 * PARTNER_WIDTH
    assert lay.width == EGO_WIDTH + 4 * PARTNER_WIDTH + 5 * ROAD_SLOT_WIDTH


def test_from_file(tmp_path):
    p = tmp_path / "sim.cfg"
    p.write_text("# engine settings\ndynamics = invertible\ngoal_tolerance = 3.5\n"
                 "collision_behavior = remove_agent\ninit_mode = all_valid\n"
                 "max_controlled_per_world = 4\nseed = 9\naccel_bounds = -3,3\nmode = lidar\n"
                 "n_rays = 32\nmax_range = 42.0\n")
    c = SimConfig.from_file(str(p))
    assert c.dynamics == "invertible" and c.goal_tolerance == 3.5
    assert c.collision_behavior == "remove_agent" and c.init_mode == "all_valid"
    assert c.max_controlled_per_world == 4 and c.seed == 9 and c.accel_bounds == (-3.0, 3.0)
    assert c.obs.mode == "lidar" and c.obs.n_rays == 32 and c.obs.max_range == 42.0
    p.write_text("bogus_key = 1\n")
    with pytest.raises(KeyError):
        SimConfig.from_file(str(p))


def test_delta_local_is_an_extension():
    c = SimConfig(dynamics="delta_local")
    assert c.action_dim == 3 and SimConfig().action_dim == 2
