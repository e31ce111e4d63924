"""make_policy / goal_seek (engine.py:535-574) on the GPU, pinned to the
reference's end-to-end acceptance scenario (test_acceptance.py:425-438):
straight_road and intersection templates, 4 agents, seed 0, driven by the
reference's own goal_seek_actions (tests/golden/templates_goal_seek.npz).

Our ds_goal_seek computes the actions from the device state each step; they
must equal the reference's (float32-rounded) actions within 2 float32 ulp
(CUDA's atan2 is not glibc's), and the episode must end as the reference's
did: every controlled agent at its goal, no collision, no off-road."""

import numpy as np
import pytest
import torch

from golden_util import load
from paper_2408_01584_b200.engine import make_policy, goal_seek_actions, benchmark

pytestmark = pytest.mark.gpu


def test_goal_seek_matches_reference_acceptance_run():
    from paper_2408_01584_b200.engine import SimBatch
    z, raw, cfg = load("templates_goal_seek")
    batch = SimBatch.from_raw(raw, cfg, device="cuda:0")
    pol = make_policy("goal_seek", cfg, batch)
    for t in range(1, z["actions"].shape[0] + 1):
        a = pol(t)
        ref = z["actions"][t - 1].astype(np.float32)
        got = a.cpu().numpy()
        tol = 2 * np.spacing(np.abs(ref)) + 1e-6
        assert (np.abs(got - ref) <= tol).all(), f"step {t}: max diff {np.abs(got - ref).max()}"
        out = batch.step(a)
        assert np.array_equal(out.rewards.cpu().numpy(), z["rewards"][t - 1].astype(np.float32))
        assert np.array_equal(out.dones.cpu().numpy(), z["dones"][t - 1])
        assert np.array_equal(batch._info[:, :batch.n_controlled].cpu().numpy(), z["info"][t - 1])
    eps = [(e.world_id, e.n_controlled, e.n_goal, e.n_veh_collision, e.n_offroad)
           for e in batch.episode_infos]
    assert np.array_equal(np.array(eps, np.int64).reshape(-1, 5), z["episodes"])
    # the acceptance criterion itself
    assert all(e[2] == e[1] and e[3] == 0 and e[4] == 0 for e in eps) and len(eps) == 2
    batch.close()


def test_make_policy_specs():
    from paper_2408_01584_b200.engine import SimBatch
    z, raw, cfg = load("templates_goal_seek")
    batch = SimBatch.from_raw(raw, cfg, device="cuda:0")
    n = batch.n_controlled
    assert make_policy("replay", cfg, batch)(0) is None
    c = make_policy("constant:1.5:-0.2", cfg, batch)(3)
    assert c.shape == (n, 2) and torch.all(c[:, 0] == 1.5) and torch.all(c[:, 1] == np.float32(-0.2))
    r = make_policy("random", cfg, batch, seed=4)(7)
    assert r.shape == (n, 2) and torch.all(r[:, 0].abs() <= 4) and torch.all(r[:, 1].abs() <= 0.7)
    g = goal_seek_actions(batch)
    assert torch.equal(g, make_policy("goal_seek", cfg, batch)(0))
    with pytest.raises(ValueError):
        make_policy("nonsense", cfg, batch)
    batch.close()


def test_benchmark_goal_seek_policy():
    from paper_2408_01584_b200.synthetic import to_scenarios
    z, raw, cfg = load("templates_goal_seek")
    rep = benchmark(to_scenarios(raw), cfg, worlds=4, steps=30, policy="goal_seek", device="cuda:0")
    assert rep.steps == 30 and rep.worlds == 4 and rep.asps > 0
