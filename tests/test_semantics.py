"""Semantics of the batched step, restated from the reference's own test suite
(pkg/tests/test_engine.py, test_observation.py) and run on both backends:
the C oracle on CPU and the CUDA engine on the GPU (marked gpu)."""

import math

import numpy as np
import pytest

from paper_2408_01584_b200.config import EGO_WIDTH, ObsConfig, SimConfig, obs_width
from paper_2408_01584_b200.scenario import RoadElement, Vec2
from scenes import Runner, hold, obs_agents, scene, scripted_object

BACKENDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


def partners(row, cfg=ObsConfig()):
    return row[EGO_WIDTH:EGO_WIDTH + 7 * cfg.max_agents_obs].reshape(cfg.max_agents_obs, 7)


def roads(row, cfg=ObsConfig()):
    off = EGO_WIDTH + 7 * cfg.max_agents_obs
    return row[off:off + 11 * cfg.max_road_points_obs].reshape(cfg.max_road_points_obs, 11)


# -- rewards, goal removal (test_engine.py:50-90) ---------------------------

@pytest.mark.parametrize("backend", BACKENDS)
def test_goal_reward_then_removal(backend):
    obj = scripted_object(0, hold(0, 0, 0.0, 5), goal=(1.9, 0.0))
    watcher = scripted_object(1, hold(0, 30.0, 0.0, 5), goal=(80, 30))
    r = Runner([scene([obj, watcher])], SimConfig(init_mode="all_valid"), backend)
    acts = np.zeros((r.n_controlled, 2))
    rew, done, info = r.step(acts)
    assert rew[0] == 1.0 and done[0] and info["goal"][0]
    assert not r.world().removed[0]
    assert (r.obs[0] == 0).all()
    rew2, done2, _ = r.step(acts)
    assert r.world().removed[0]
    assert rew2[0] == 0.0 and done2[0]
    assert partners(r.obs[1])[0, 6] == 0.0      # the watcher lost its partner
    r.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_cumulative_reward_at_most_one(backend):
    obj = scripted_object(0, hold(0, 0, 0.0, 6), goal=(0.5, 0.0))
    r = Runner([scene([obj])], SimConfig(init_mode="all_valid"), backend)
    total = sum(r.step(np.zeros((1, 2)))[0][0] for _ in range(5))
    assert total == 1.0
    r.close()


# -- collisions (test_engine.py:97-192) -------------------------------------

def head_on(extra=()):
    a = scripted_object(0, hold(-1.0, 0, 0.0, 5), goal=(50, 0))
    b = scripted_object(1, hold(1.0, 0, math.pi, 5), goal=(-50, 0))
    return [a, b, *extra]


@pytest.mark.parametrize("backend", BACKENDS)
def test_head_on_collision_remove_agent(backend):
    r = Runner([scene(head_on())], SimConfig(collision_behavior="remove_agent"), backend)
    _, done, info = r.step(np.zeros((2, 2)))
    assert info["veh_collision"].tolist() == [True, True]
    assert done.tolist() == [True, True]
    r.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_collision_ignore_keeps_agents_alive(backend):
    r = Runner([scene(head_on())], SimConfig(collision_behavior="ignore"), backend)
    _, done, info = r.step(np.zeros((2, 2)))
    assert info["veh_collision"].tolist() == [True, True]
    assert done.tolist() == [False, False]
    r.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_collision_end_episode_finishes_world(backend):
    c = scripted_object(2, hold(0.0, 30, 0.0, 5), goal=(50, 30))
    r = Runner([scene(head_on([c]))], SimConfig(collision_behavior="end_episode"), backend)
    _, done, _ = r.step(np.zeros((3, 2)))
    assert done.tolist() == [True, True, True]
    assert r.world().episode_over
    r.close()


EDGE = RoadElement(id=0, kind="road_edge", geometry=[Vec2(5.0, -10), Vec2(5.0, 10)])


@pytest.mark.parametrize("backend", BACKENDS)
def test_pedestrian_road_edge_exemption(backend):
    ped = scripted_object(0, hold(5.0, 0, 0.0, 4), kind="pedestrian", goal=(30, 0),
                          length=0.8, width=0.8)
    veh = scripted_object(1, hold(5.0, 5.0, 0.0, 4), goal=(30, 5))
    r = Runner([scene([ped, veh], [EDGE])], SimConfig(), backend)
    _, _, info = r.step(np.zeros((2, 2)))
    assert not info["offroad"][0] and info["offroad"][1]
    r.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_cyclist_hits_edge_and_lanes_do_not(backend):
    cyc = scripted_object(0, hold(5.0, 0, 0.0, 4), kind="cyclist", goal=(30, 0), length=1.8,
                          width=0.6)
    r = Runner([scene([cyc], [EDGE])], SimConfig(), backend)
    assert r.step(np.zeros((1, 2)))[2]["offroad"][0]
    r.close()
    lane = RoadElement(id=0, kind="lane", geometry=[Vec2(5.0, -10), Vec2(5.0, 10)])
    veh = scripted_object(0, hold(5.0, 0, 0.0, 4), goal=(30, 0))
    r = Runner([scene([veh], [lane])], SimConfig(), backend)
    assert not r.step(np.zeros((1, 2)))[2]["offroad"][0]
    r.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_removed_agent_not_in_collisions(backend):
    a = scripted_object(0, hold(0, 0, 0.0, 6), goal=(0.0, 0.0))
    b = scripted_object(1, [(-8.0 + 2.0 * t, 0.0, 0.0) for t in range(6)], goal=(100, 0),
                        force_replay=True)
    r = Runner([scene([a, b])], SimConfig(init_mode="all_valid"), backend)
    assert r.step(np.zeros((1, 2)))[0][0] == 1.0
    for _ in range(4):
        assert not r.step(np.zeros((1, 2)))[2]["veh_collision"][0]
    r.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_invalid_replay_steps_hold_pose_and_skip_collision(backend):
    ghost = scripted_object(1, [(20.0, 0, 0.0)] * 5, goal=(20, 0), force_replay=True,
                            valid=[True, True, False, False, True])
    mover = scripted_object(0, [(18.0 + t, 0, 0.0) for t in range(5)], goal=(60, 0))
    r = Runner([scene([mover, ghost])], SimConfig(), backend)
    acts = np.zeros((1, 2))
    assert r.step(acts)[2]["veh_collision"][0]
    assert not r.step(acts)[2]["veh_collision"][0]
    assert r.world().pos[1, 0] == 20.0
    assert not r.step(acts)[2]["veh_collision"][0]
    assert r.step(acts)[2]["veh_collision"][0]
    r.close()


# -- initialisation modes (test_engine.py:232-272) --------------------------

@pytest.mark.parametrize("backend", BACKENDS)
def test_init_modes(backend):
    parked = scripted_object(0, hold(0, 0, 0.0, 3), goal=(1.0, 0.0))
    mover = scripted_object(1, hold(10, 0, 0.0, 3), goal=(50.0, 0.0))
    r = Runner([scene([parked, mover])], SimConfig(init_mode="all_nontrivial"), backend)
    assert r.world().controlled_ids.tolist() == [1]
    r.close()
    r = Runner([scene([parked, mover])], SimConfig(init_mode="all_valid"), backend)
    assert r.world().controlled_ids.tolist() == [0, 1]
    r.close()
    objs = [scripted_object(i, hold(10.0 * i, 0, 0.0, 3), goal=(10.0 * i + 30, 0))
            for i in range(6)]
    r = Runner([scene(objs)], SimConfig(max_controlled_per_world=3), backend)
    assert r.world().controlled_ids.tolist() == [0, 1, 2]
    r.close()
    forced = scripted_object(0, hold(0, 0, 0.0, 3), goal=(50, 0.0), force_replay=True)
    for mode in ("all_nontrivial", "all_valid"):
        r = Runner([scene([forced, mover])], SimConfig(init_mode=mode), backend)
        assert 0 not in r.world().controlled_ids.tolist()
        r.close()


# -- replay, horizon, reset (test_engine.py:279-320) ------------------------

@pytest.mark.parametrize("backend", BACKENDS)
def test_replay_reproduces_logged_poses_and_horizon(backend):
    objs = [scripted_object(i, [(3.0 * t + i, 0.5 * t * i, 0.01 * t) for t in range(9)],
                            valid=[True] * 4 + [False] + [True] * 4) for i in range(3)]
    prep = scene(objs)
    r = Runner([prep], SimConfig(init_mode="all_valid"), backend)
    for t in range(1, 9):
        _, done, _ = r.step(None)
        assert r.world().t == t
        for i, o in enumerate(prep.base.objects):
            st = o.states[t]
            if st.valid:
                assert r.world().pos[i, 0] == st.position.x
                assert r.world().pos[i, 1] == st.position.y
                assert r.world().heading[i] == st.heading
    _, done, _ = r.step(None)
    assert r.world().episode_over and done.all()
    r.reset()
    assert r.world().t == 0 and not r.world().episode_over
    assert not r.world().done.any() and not r.world().removed.any()
    r.close()


# -- batch (test_engine.py:344-432) -------------------------------------------

@pytest.mark.parametrize("backend", BACKENDS)
def test_identical_worlds_identical_and_partial_reset(backend):
    objs = [scripted_object(i, [(3.0 * t + 5 * i, 2.0 * i, 0.0) for t in range(12)],
                            goal=(40 + 5 * i, 2.0 * i)) for i in range(4)]
    edge = RoadElement(id=0, kind="road_edge", geometry=[Vec2(-10, -3), Vec2(80, -3)])
    prep = scene(objs, [edge])
    r = Runner([prep] * 4, SimConfig(), backend)
    per = r.n_controlled // 4
    rng = np.random.default_rng(3)
    for _ in range(6):
        acts = np.tile(rng.uniform(-1, 1, (per, 2)), (4, 1))
        r.step(acts)
        obs = r.obs
        for k in range(1, 4):
            assert (obs[k * per:(k + 1) * per] == obs[:per]).all()
    before = r.obs.copy()
    t_before = [r.world(w).t for w in range(4)]
    r.reset([2])
    assert [r.world(w).t for w in range(4)] == [t_before[0], t_before[1], 0, t_before[3]]
    outside = np.ones(r.n_controlled, bool)
    outside[2 * per:3 * per] = False
    assert (r.obs[outside] == before[outside]).all()
    r.close()


# -- head rotation (test_engine.py:583-592) ---------------------------------

@pytest.mark.parametrize("backend", BACKENDS)
def test_head_rotation_integrates_and_clamps(backend):
    obj = scripted_object(0, hold(0, 0, 0.0, 40), goal=(100, 0))
    cfg = SimConfig(obs=ObsConfig(mode="view_cone", n_rays=8))
    r = Runner([scene([obj])], cfg, backend)
    acts = np.array([[0.0, 0.0, 1.0]])
    r.step(acts)
    assert abs(r.world().head_angle[0] - 0.1) < 1e-12
    for _ in range(30):
        r.step(acts)
    assert r.world().head_angle[0] == pytest.approx(math.pi / 2)
    r.close()


# -- radial observations (test_observation.py:37-110, 306-325) --------------

def radial_obs(agents, backend, cfg=ObsConfig(), roads_=()):
    r = Runner([obs_agents(agents, roads_)], SimConfig(obs=cfg, init_mode="all_valid"), backend)
    row = r.obs[0].copy()
    r.close()
    return row


@pytest.mark.parametrize("backend", BACKENDS)
def test_lone_agent_empty_map(backend):
    row = radial_obs([(0.0, 0.0, 0.0, 5.0, "vehicle", 4.0, 2.0, (30.0, 40.0))], backend)
    assert row[0] == 5.0 and row[3] == 30.0 and row[4] == 40.0 and row[5] == 50.0
    assert (partners(row) == 0).all() and (roads(row) == 0).all()


@pytest.mark.parametrize("backend", BACKENDS)
def test_radius_threshold_semantics(backend):
    assert partners(radial_obs([(0, 0, 0, 0), (51.0, 0, 0, 0)], backend))[0, 6] == 0.0
    p = partners(radial_obs([(0, 0, 0, 0), (49.0, 0, 0, 0)], backend))
    assert p[0, 6] == 1.0 and abs(p[0, 0] - 49.0) < 1e-12
    p = partners(radial_obs([(0, 0, 0, 0), (50.0, 0, 0, 0)], backend))   # exactly on the radius
    assert p[0, 6] == 1.0


@pytest.mark.parametrize("backend", BACKENDS)
def test_partner_cap_keeps_nearest(backend):
    cfg = ObsConfig(mode="radial", radius=200.0, max_agents_obs=16)
    rng = np.random.default_rng(0)
    agents = [(0.0, 0.0, 0.0, 0.0)] + [(float(rng.uniform(-80, 80)), float(rng.uniform(-80, 80)),
                                        0.0, 0.0) for _ in range(30)]
    p = partners(radial_obs(agents, backend, cfg), cfg)
    dists = sorted(math.hypot(a[0], a[1]) for a in agents[1:])[:16]
    got = [math.hypot(p[k, 0], p[k, 1]) for k in range(16)]
    assert np.allclose(got, dists, atol=1e-4)
    assert (p[:, 6] == 1).all()


@pytest.mark.parametrize("backend", BACKENDS)
def test_equal_distance_ties_keep_smaller_index(backend):
    """Four partners at exactly the same distance: slots in index order."""
    cfg = ObsConfig(mode="radial", max_agents_obs=3)
    agents = [(0.0, 0.0, 0.0, 0.0), (0.0, 10.0, 0.0, 1.0), (10.0, 0.0, 0.0, 2.0),
              (-10.0, 0.0, 0.0, 3.0), (0.0, -10.0, 0.0, 4.0)]
    p = partners(radial_obs(agents, backend, cfg), cfg)
    assert p[:, 3].tolist() == [1.0, 2.0, 3.0]     # relative speeds identify agents 1, 2, 3


@pytest.mark.parametrize("backend", BACKENDS)
def test_partner_slots_relative_frame(backend):
    p = partners(radial_obs([(10, 5, math.pi / 2, 2.0), (10, 8, math.pi / 2, 6.0)], backend))
    assert abs(p[0, 0] - 3.0) < 1e-12 and abs(p[0, 1]) < 1e-12 and abs(p[0, 2]) < 1e-12
    assert abs(p[0, 3] - 4.0) < 1e-12 and p[0, 4] == 4.0 and p[0, 5] == 2.0


@pytest.mark.parametrize("backend", BACKENDS)
def test_road_points_relative_and_typed(backend):
    cfg = ObsConfig(mode="radial", max_road_points_obs=8)
    road = RoadElement(id=0, kind="road_edge", geometry=[Vec2(2, -1), Vec2(10, -1)])
    rd = roads(radial_obs([(0, 0, 0.0, 0.0)], backend, cfg, [road]), cfg)
    assert rd[0, -1] == 1.0 and abs(rd[0, 0] - 2.0) < 1e-12 and abs(rd[0, 1] + 1.0) < 1e-12
    assert rd[0, 3] == 1.0
    assert rd[1, -1] == 1.0 and abs(rd[1, 0] - 10.0) < 1e-12
    assert (rd[2:] == 0).all()


def _scene(dx=0.0, dy=0.0, rot=0.0):
    c, s = math.cos(rot), math.sin(rot)

    def move(x, y):
        return (x * c - y * s + dx, x * s + y * c + dy)

    agents = []
    for (x, y, h, v) in [(0, 0, 0.2, 3.0), (8, 2, -1.0, 5.0), (-4, 6, 2.0, 1.0)]:
        mx, my = move(x, y)
        agents.append((mx, my, h + rot, v, "vehicle", 4.0, 2.0, move(x + 20, y)))
    road = RoadElement(id=0, kind="road_edge", geometry=[Vec2(*move(-10, -5)),
                                                          Vec2(*move(15, -5)),
                                                          Vec2(*move(15, 10))])
    return agents, [road]


@pytest.mark.parametrize("backend", BACKENDS)
def test_translation_and_rotation_invariance(backend):
    base = radial_obs(*_scene()[:1], backend, ObsConfig(), _scene()[1])
    for kw in (dict(dx=137.0, dy=-64.0), dict(rot=0.83)):
        a, rd = _scene(**kw)
        other = radial_obs(a, backend, ObsConfig(), rd)
        assert np.allclose(base, other, atol=1e-4)


# -- LiDAR / view cone (test_observation.py:161-281) ------------------------

LIDAR_BACKENDS = BACKENDS


@pytest.mark.parametrize("backend", LIDAR_BACKENDS)
def test_lidar_wall_ahead_four_rays(backend):
    cfg = ObsConfig(mode="lidar", n_rays=4, max_range=100.0)
    row = radial_obs([(0, 0, 0.0, 0.0)], backend, cfg, [EDGE])
    rays = row[EGO_WIDTH:].reshape(4, 5)
    assert rays[0, 0] == 5.0 and rays[0, 2] == 1.0
    for k in (1, 2, 3):
        assert rays[k, 0] == 100.0 and rays[k, 4] == 1.0


@pytest.mark.parametrize("backend", LIDAR_BACKENDS)
def test_lidar_empty_world_and_ego_excluded(backend):
    cfg = ObsConfig(mode="lidar", n_rays=8)
    rays = radial_obs([(3, 4, 1.0, 0.0, "vehicle", 6.0, 3.0)], backend, cfg)[EGO_WIDTH:]
    rays = rays.reshape(8, 5)
    assert (rays[:, 0] == cfg.max_range).all() and (rays[:, 4] == 1.0).all()


@pytest.mark.parametrize("backend", LIDAR_BACKENDS)
def test_view_cone_behind_not_visible(backend):
    cfg = ObsConfig(mode="view_cone", n_rays=31, fov=2 * math.pi / 3, max_range=50.0)
    rays = radial_obs([(0, 0, 0.0, 0.0), (-7.0, 7.0, 0.0, 0.0)], backend, cfg)[EGO_WIDTH:]
    assert (rays.reshape(31, 5)[:, 0] == cfg.max_range).all()
