"""GPU parity: the CUDA step (through the C ABI) against the C oracle, which is
itself pinned bit-exact to the reference (tests/test_oracle_golden.py).

Free-run over a full 91-step episode: rewards, dones, info flags and the
partner / road-point selection indices must be bit-exact; observations within
2 float32 ulp + 1e-6 of the FP64 oracle rounded to float32; poses within
1e-9 m / 1e-12 rad (FP64 state; only transcendental ulps differ).  Every
case runs on the benchmark's 2^-10 m lattice AND off it (full FP64
coordinates, so the float32 copies the kernels cull with carry a rounding
error: the grid_eps term of the key bound is live).
"""

import numpy as np
import pytest
import torch

from paper_2408_01584_b200.config import ObsConfig, SimConfig
from paper_2408_01584_b200.engine import SimBatch
from paper_2408_01584_b200.synthetic import WaymoSpec, generate
from oracle.oracle import OracleBatch
from parity import ANG_TOL, POS_TOL, actions_for, compare_step, wrap_diff

pytestmark = pytest.mark.gpu

CASES = {
    "c1_classic_remove": (dict(n_worlds=8, n_agents=32, n_points=400),
                          dict(collision_behavior="remove_agent")),
    "c1_invertible_ignore": (dict(n_worlds=8, n_agents=32, n_points=400),
                             dict(dynamics="invertible")),
    "c1_end_episode": (dict(n_worlds=8, n_agents=32, n_points=400),
                       dict(collision_behavior="end_episode")),
    "c1_delta_local": (dict(n_worlds=8, n_agents=32, n_points=400),
                       dict(dynamics="delta_local", collision_behavior="remove_agent")),
    "c2_shape": (dict(n_worlds=12, n_agents=64, n_points=2000),
                 dict(collision_behavior="remove_agent")),
    "c3_shape": (dict(n_worlds=3, n_agents=128, n_points=10000),
                 dict(dynamics="delta_local")),
    "small_caps": (dict(n_worlds=6, n_agents=40, n_points=900),
                   dict(obs=ObsConfig(max_agents_obs=3, max_road_points_obs=5, radius=30.0))),
    "big_caps": (dict(n_worlds=4, n_agents=100, n_points=6000),
                 dict(obs=ObsConfig(max_agents_obs=128, max_road_points_obs=128, radius=80.0))),
    # >= 2 x 148 worlds of <= 64 agents: the two-CTAs-per-SM observation variant
    "many_small_worlds": (dict(n_worlds=300, n_agents=24, n_points=300),
                          dict(collision_behavior="remove_agent")),
    # 129..256 agents: the 256-thread step kernel variant
    "agents_200": (dict(n_worlds=3, n_agents=200, n_points=2000),
                   dict(collision_behavior="remove_agent")),
    # 13k points: the shared-point kernel with 24 warps (32 do not fit)
    "mid_world": (dict(n_worlds=2, n_agents=48, n_points=13000),
                  dict(collision_behavior="remove_agent")),
    # > shared-memory capacity: exercises the global-memory point scan
    "huge_world": (dict(n_worlds=2, n_agents=48, n_points=32000),
                   dict(collision_behavior="remove_agent")),
}


def _gpu_out(batch):
    return {"obs": batch.observations.cpu().numpy(), "rewards": batch.rewards.cpu().numpy(),
            "dones": batch.dones.cpu().numpy(), "info": batch._info[:, :batch.n_controlled].cpu().numpy()}


def run_free(case, steps=91, seed=0, raw=None, cfg=None, quantize=True):
    if raw is None:
        spec_kw, cfg_kw = CASES[case]
        cfg = SimConfig(init_mode="all_valid", **cfg_kw)
        raw = generate(WaymoSpec(seed=seed + 11, quantize=quantize, **spec_kw))
    lidar = cfg.obs.mode != "radial"
    batch = SimBatch.from_raw(raw, cfg, device="cuda:0")
    OracleBatch.lidar_ties()                 # reset the tie counter
    ora = OracleBatch(raw, cfg)
    n = batch.n_controlled
    sel_w = cfg.obs.max_agents_obs + cfg.obs.max_road_points_obs
    sel = None if lidar else torch.full((n, sel_w), -7, dtype=torch.int32, device="cuda:0")
    batch.reset(sel_idx=sel)
    sel_of = (lambda: None) if lidar else (lambda: sel.cpu().numpy())
    ora_sel = (lambda: None) if lidar else (lambda: ora.sel_idx[:n])
    compare_step(0, _gpu_out(batch), (ora.observations, ora.rewards, ora.dones.astype(bool),
                                      {k: np.zeros(n, bool) for k in ("goal", "veh_collision", "offroad")}),
                 sel_of(), ora_sel())
    rng = np.random.default_rng(seed)
    for t in range(1, steps + 1):
        act = actions_for(cfg, n, rng)
        batch.step(torch.from_numpy(act).cuda(), sel_idx=sel)
        o = ora.step(act.astype(np.float64))
        compare_step(t, _gpu_out(batch), o, sel_of(), ora_sel())
    pw = batch.packed
    x, y, h = batch._x.cpu().numpy(), batch._y.cpu().numpy(), batch._h.cpu().numpy()
    nA = pw.n_agents
    assert np.abs(x[:nA] - ora.x[:nA]).max() <= POS_TOL
    assert np.abs(y[:nA] - ora.y[:nA]).max() <= POS_TOL
    assert wrap_diff(h[:nA], ora.heading[:nA]).max() <= ANG_TOL
    assert np.array_equal(batch._flags.cpu().numpy()[:nA].astype(np.uint16), ora.flags[:nA])
    eps = [(e.world_id, e.n_controlled, e.n_goal, e.n_veh_collision, e.n_offroad)
           for e in batch.episode_infos]
    assert eps == ora.episode_infos
    # edge / non-edge exact ties (reference: BVH order; here: edge first)
    assert OracleBatch.lidar_ties() == 0
    batch.close()


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("lattice", ["lattice", "offlattice"])
def test_free_run_parity(case, lattice):
    run_free(case, quantize=lattice == "lattice")


def test_replay_mode_parity():
    """actions=None: expert replay for everyone (engine.py:383-385)."""
    cfg = SimConfig(init_mode="all_valid")
    raw = generate(WaymoSpec(n_worlds=4, n_agents=32, n_points=400, seed=5))
    batch = SimBatch.from_raw(raw, cfg, device="cuda:0")
    ora = OracleBatch(raw, cfg)
    for t in range(1, 92):
        batch.step(None)
        o = ora.step(None)
        compare_step(t, _gpu_out(batch), o)
    assert np.array_equal(batch._x.cpu().numpy(), ora.x)   # replay copies poses bit-exactly
    batch.close()


def test_auto_reset_env_semantics():
    """auto_reset: finished worlds reset in-kernel, rewards rows zeroed (env.py:95-109)."""
    cfg = SimConfig(init_mode="all_valid", collision_behavior="end_episode")
    raw = generate(WaymoSpec(n_worlds=6, n_agents=32, n_points=400, seed=9))
    batch = SimBatch.from_raw(raw, cfg, device="cuda:0")
    ora = OracleBatch(raw, cfg)
    rng = np.random.default_rng(3)
    for t in range(1, 200):
        act = actions_for(cfg, batch.n_controlled, rng)
        batch.step(torch.from_numpy(act).cuda(), auto_reset=True)
        o = ora.step(act.astype(np.float64), auto_reset=True)
        compare_step(t, _gpu_out(batch), o)
    eps = [(e.world_id, e.n_controlled, e.n_goal, e.n_veh_collision, e.n_offroad)
           for e in batch.episode_infos]
    assert eps == ora.episode_infos and len(eps) > 6
    batch.close()


@pytest.mark.parametrize("quantize", [True, False])
@pytest.mark.parametrize("init_mode", ["all_nontrivial", "all_valid"])
def test_ragged_batch_parity(init_mode, quantize):
    """Worlds of 1..300 agents and 0..5000 road points, late entries, blink-outs,
    never-valid and forced-replay agents, single-point road elements, agents
    far off the map (tests/ragged.py)."""
    from ragged import ragged_batch
    cfg = SimConfig(init_mode=init_mode, collision_behavior="remove_agent",
                    max_controlled_per_world=250)
    run_free(None, raw=ragged_batch(seed=3, quantize=quantize), cfg=cfg)


@pytest.mark.parametrize("quantize", [True, False])
def test_ragged_batch_lidar_parity(quantize):
    from ragged import ragged_batch
    cfg = SimConfig(init_mode="all_valid", obs=ObsConfig(mode="lidar", n_rays=24, max_range=60.0))
    run_free(None, raw=ragged_batch(seed=4, num_steps=30, quantize=quantize), cfg=cfg, steps=30)


@pytest.mark.parametrize("quantize", [True, False])
def test_lidar_c4_shape_parity(quantize):
    """BASELINE config 4 shape (128 agents, 10k points, 64 rays, 50 m) on two
    worlds over a full 91-step episode: the grid-ring / occlusion-culled
    kernel against the oracle's brute force over all boxes and segments."""
    cfg = SimConfig(init_mode="all_valid", obs=ObsConfig(mode="lidar", n_rays=64, max_range=50.0))
    raw = generate(WaymoSpec(n_worlds=2, n_agents=128, n_points=10000, seed=21, quantize=quantize))
    run_free(None, raw=raw, cfg=cfg, steps=91)


def test_lidar_delta_local_remove_agent_parity():
    """LiDAR with delta-local dynamics (3 action columns) and removal."""
    cfg = SimConfig(init_mode="all_valid", dynamics="delta_local", collision_behavior="remove_agent",
                    obs=ObsConfig(mode="lidar", n_rays=40, max_range=35.0))
    raw = generate(WaymoSpec(n_worlds=4, n_agents=48, n_points=3000, seed=31))
    run_free(None, raw=raw, cfg=cfg, steps=40)


def test_view_cone_parity_with_head_rotation():
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent",
                    obs=ObsConfig(mode="view_cone", n_rays=17, fov=2.5, max_range=70.0))
    raw = generate(WaymoSpec(n_worlds=4, n_agents=40, n_points=1500, seed=8))
    batch = SimBatch.from_raw(raw, cfg, device="cuda:0")
    ora = OracleBatch(raw, cfg)
    rng = np.random.default_rng(2)
    for t in range(1, 40):
        act = actions_for(cfg, batch.n_controlled, rng, head=True)
        batch.step(torch.from_numpy(act).cuda())
        compare_step(t, _gpu_out(batch), ora.step(act.astype(np.float64)))
    batch.close()
