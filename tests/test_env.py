"""VecDriveEnv drop-in (pkg/rl/src/drivesim_rl/env.py), restating the
reference's env tests (pkg/rl/tests/test_env.py) on the GPU engine, with the
C oracle (driven through the same continuous actions and auto-reset) as the
checker."""

import math

import numpy as np
import pytest
import torch

from paper_2408_01584_b200.config import ObsConfig, SimConfig, obs_width
from paper_2408_01584_b200.env import ActionGrid, EnvConfig, IndexOutOfRange, obs_scale
from paper_2408_01584_b200.synthetic import WaymoSpec, generate
from parity import obs_tolerance


def small_obs():
    return ObsConfig(max_agents_obs=8, max_road_points_obs=16)


def test_action_grid_round_trip():
    g = ActionGrid()
    assert g.size == 91
    for k in range(g.size):
        a, s = g.discretize(k)
        assert g.action_index(a, s) == k
    with pytest.raises(IndexOutOfRange):
        g.discretize(91)
    with pytest.raises(ValueError):
        ActionGrid(accelerations=[1.0, 0.0])


def test_env_config_validation():
    with pytest.raises(ValueError):
        EnvConfig(rollout_length=0)
    assert EnvConfig().sim.collision_behavior == "remove_agent"


def test_obs_scale_layout():
    s = obs_scale(SimConfig(obs=small_obs()))
    assert s.shape == (obs_width(small_obs()),)
    assert s[0] == 100.0 and s[3] == 50.0 and s[7 + 2] == math.pi


@pytest.mark.gpu
def test_env_matches_oracle_with_auto_reset():
    from oracle.oracle import OracleBatch
    from paper_2408_01584_b200.env import VecDriveEnv
    from paper_2408_01584_b200.packing import pack
    raw = generate(WaymoSpec(n_worlds=5, n_agents=24, n_points=500, seed=13, num_steps=20))
    sim = SimConfig(collision_behavior="remove_agent", obs=small_obs(), init_mode="all_valid")
    env = VecDriveEnv(EnvConfig(raw=raw, sim=sim, device="cuda:0"))
    ora = OracleBatch(raw, sim)
    scale = obs_scale(sim)
    obs = env.reset().cpu().numpy()
    assert obs.shape == (env.n_agents, env.obs_width)
    ref = ora.observations / scale
    assert (np.abs(obs - ref.astype(np.float32)) <= obs_tolerance(ref)).all()
    rng = np.random.default_rng(0)
    episodes = 0
    for t in range(45):                          # crosses two auto-resets
        idx = rng.integers(0, env.n_actions, env.n_agents)
        obs, rew, done, infos = env.step(torch.from_numpy(idx).cuda())
        cont = env.to_continuous(idx).cpu().numpy()
        o_obs, o_rew, o_done, o_info = ora.step(cont, auto_reset=True)
        assert np.array_equal(rew.cpu().numpy(), o_rew.astype(np.float32))
        assert np.array_equal(done.cpu().numpy(), o_done)
        for k in ("goal", "veh_collision", "offroad"):
            assert np.array_equal(infos[k].cpu().numpy(), o_info[k])
        ref = o_obs / scale
        err = np.abs(obs.cpu().numpy().astype(np.float64) - ref.astype(np.float32))
        assert (err <= obs_tolerance(ref)).all(), f"t={t} max err {err.max()}"
        episodes += len(infos["episodes"])
    assert episodes == 2 * 5 == len(ora.episode_infos)
    env.close()


@pytest.mark.gpu
def test_inverted_expert_actions_reach_all_goals():
    """RT/test_env.py:104-129: actions inverted from the (straight, constant
    speed) expert logs under invertible dynamics reach every goal."""
    from paper_2408_01584_b200.env import VecDriveEnv
    from scenes import scene, scripted_object
    T, dt = 91, 0.1
    scenes = []
    for s_ in range(3):
        objs = [scripted_object(i, [(-12.0 * i + (4.0 + s_) * dt * t, 4.0 * (i % 4), 0.0)
                                    for t in range(T)], speed=4.0 + s_) for i in range(4)]
        scenes.append(scene(objs))
    sim = SimConfig(dynamics="invertible", collision_behavior="ignore", obs=small_obs())
    env = VecDriveEnv(EnvConfig(scenarios=scenes, num_worlds=3, sim=sim, normalize_obs=False,
                                device="cuda:0"))
    env.reset()
    worlds = env.batch.worlds
    n_goal = n_ctrl = 0
    for t in range(T):
        acts = []
        for w in worlds:
            ids = w.controlled_ids
            t1 = min(t + 1, w.num_steps - 1)
            h0, v0 = w.replay_heading[ids, t], w.replay_speed[ids, t]
            h1, v1 = w.replay_heading[ids, t1], w.replay_speed[ids, t1]
            a = (v1 - v0) / w.dt
            den = v0 * w.dt + 0.5 * a * w.dt * w.dt
            dth = np.mod(h1 - h0 + math.pi, 2 * math.pi) - math.pi
            s = np.where(np.abs(den) < 1e-9, 0.0, dth / np.where(den == 0, 1, den))
            acts.append(np.column_stack([a, s]))
        _, _, _, infos = env.step(torch.from_numpy(np.vstack(acts)).float().cuda())
        for e in infos["episodes"]:
            n_goal += e.n_goal
            n_ctrl += e.n_controlled
    assert n_ctrl > 0 and n_goal == n_ctrl
    env.close()


@pytest.mark.gpu
def test_out_of_grid_action_index_raises():
    """to_continuous (env.py:111-116) indexes numpy arrays: a joint index in
    [-91, 91) is valid (negative ones count from the end), anything else
    raises IndexError -- never a silently clamped action."""
    from paper_2408_01584_b200.env import VecDriveEnv
    raw = generate(WaymoSpec(n_worlds=2, n_agents=8, n_points=200, seed=2, num_steps=20))
    env = VecDriveEnv(EnvConfig(raw=raw, sim=SimConfig(obs=small_obs(), init_mode="all_valid"),
                                device="cuda:0"))
    env.reset()
    n = env.n_agents
    with pytest.raises(IndexError):
        env.step(torch.full((n,), 91))                  # host indices: checked at once
    with pytest.raises(IndexError):
        env.step(np.full(n, -92))
    env.step(torch.full((n,), -91, device="cuda:0"))    # valid: accel[-7], steer[0]
    env.batch.check_status()
    x0 = env.batch._x.clone()
    env.step(torch.full((n,), 500, device="cuda:0"))    # device indices: flagged by the kernel
    with pytest.raises(IndexError):
        env.batch.check_status()
    env.batch.check_status()                            # the flag was cleared
    env.close()


@pytest.mark.gpu
def test_kernel_arguments_are_validated():
    from paper_2408_01584_b200.engine import SimBatch
    raw = generate(WaymoSpec(n_worlds=2, n_agents=8, n_points=200, seed=2))
    cfg = SimConfig(init_mode="all_valid")
    b = SimBatch.from_raw(raw, cfg, device="cuda:0")
    act = torch.zeros((b.n_controlled, 2), device="cuda:0")
    sel_w = cfg.obs.max_agents_obs + cfg.obs.max_road_points_obs
    with pytest.raises(ValueError):          # wrong dtype
        b.step(act, sel_idx=torch.zeros((b.n_controlled, sel_w), dtype=torch.int64, device="cuda:0"))
    with pytest.raises(ValueError):          # too short
        b.step(act, sel_idx=torch.zeros((1, sel_w), dtype=torch.int32, device="cuda:0"))
    with pytest.raises(ValueError):          # host tensor
        b.step(act, obs_scale=torch.ones(b.width))
    with pytest.raises(ValueError):
        b.reset(world_mask=torch.ones(1, dtype=torch.uint8, device="cuda:0"))
    b.step(act, obs_scale=torch.ones(b.width, dtype=torch.float64, device="cuda:0"))  # converted
    b.close()
