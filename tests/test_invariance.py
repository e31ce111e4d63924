"""Properties the exact kernels must have independent of how the work is laid
out (the reference pins the same for its worker pool, T/test_engine.py:344-406):

* a world stepped inside a batch gives bit-identical rows to the same world
  stepped alone (no cross-world state, no dependence on the world's slot);
* the road grid is only an acceleration structure: observations, rewards and
  flags are bit-identical for different grid cell sizes (the culling only
  ever keeps supersets, the selection is exact);
* the same for the LiDAR grid walk.
"""

import numpy as np
import pytest
import torch

from paper_2408_01584_b200.config import ObsConfig, SimConfig
from paper_2408_01584_b200.engine import SimBatch
from paper_2408_01584_b200.packing import concat_raw
from paper_2408_01584_b200.synthetic import WaymoSpec, generate
from parity import actions_for

pytestmark = pytest.mark.gpu


def _outputs(batch):
    torch.cuda.synchronize()
    return (batch.observations.cpu().numpy().copy(), batch.rewards.cpu().numpy().copy(),
            batch.dones.cpu().numpy().copy(), batch._info[:, :batch.n_controlled].cpu().numpy().copy())


def _run(batch, acts):
    outs = []
    for a in acts:
        batch.step(torch.from_numpy(a).cuda(), auto_reset=True)
        outs.append(_outputs(batch))
    return outs


def test_world_in_batch_equals_world_alone():
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent")
    raws = [generate(WaymoSpec(n_worlds=1, n_agents=40, n_points=1500, seed=s)) for s in range(5)]
    full = SimBatch.from_raw(concat_raw(raws), cfg, device="cuda:0")
    rng = np.random.default_rng(1)
    acts = [actions_for(cfg, full.n_controlled, rng).astype(np.float32) for _ in range(30)]
    outs = _run(full, acts)
    off = full.offsets
    for w in (0, 3):
        solo = SimBatch.from_raw(raws[w], cfg, device="cuda:0")
        s_outs = _run(solo, [a[off[w]:off[w + 1]] for a in acts])
        for (o, r, d, i), (so, sr, sd, si) in zip(outs, s_outs):
            sl = slice(off[w], off[w + 1])
            assert np.array_equal(o[sl], so)
            assert np.array_equal(r[sl], sr) and np.array_equal(d[sl], sd)
            assert np.array_equal(i[:, sl], si)
        solo.close()
    full.close()


@pytest.mark.parametrize("mode,cells", [("radial", (8.0, 5.0, 13.0)), ("lidar", (10.0, 6.0, 17.0))])
def test_grid_cell_size_does_not_change_results(mode, cells):
    obs = ObsConfig() if mode == "radial" else ObsConfig(mode="lidar", n_rays=48, max_range=45.0)
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent", obs=obs)
    raw = generate(WaymoSpec(n_worlds=3, n_agents=64, n_points=4000, seed=9))
    rng = np.random.default_rng(2)
    base = None
    for cs in cells:
        b = SimBatch.from_raw(raw, cfg, device="cuda:0", grid_cell=cs)
        if base is None:
            acts = [actions_for(cfg, b.n_controlled, rng).astype(np.float32) for _ in range(12)]
        outs = _run(b, acts)
        b.close()
        if base is None:
            base = outs
            continue
        for (o, r, d, i), (bo, br, bd, bi) in zip(outs, base):
            assert np.array_equal(o, bo), f"cell {cs}: observations differ"
            assert np.array_equal(r, br) and np.array_equal(d, bd) and np.array_equal(i, bi)


def test_full_circle_view_cone_equals_lidar():
    """A view cone with fov = 2 pi and no head rotation is the LiDAR sweep
    (observation.py:213-220; T/test_observation.py:243-250)."""
    import math
    raw = generate(WaymoSpec(n_worlds=3, n_agents=40, n_points=3000, seed=13))
    outs = []
    for obs in (ObsConfig(mode="lidar", n_rays=36, max_range=40.0),
                ObsConfig(mode="view_cone", n_rays=36, fov=2 * math.pi, max_range=40.0)):
        cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent", obs=obs)
        b = SimBatch.from_raw(raw, cfg, device="cuda:0")
        rng = np.random.default_rng(4)
        acts = [actions_for(cfg, b.n_controlled, rng).astype(np.float32) for _ in range(15)]
        outs.append(_run(b, acts))
        b.close()
    for (o1, r1, d1, i1), (o2, r2, d2, i2) in zip(*outs):
        assert np.array_equal(o1, o2)
        assert np.array_equal(r1, r2) and np.array_equal(d1, d2) and np.array_equal(i1, i2)


@pytest.mark.parametrize("hint", ["bogus_small", "bogus_large", "none"])
def test_search_hint_never_changes_results(hint):
    """The radial search hint (last step's k-th distance bound and position)
    only narrows a provably sufficient disc: a deliberately wrong hint -- far
    too small (the narrowed histogram's validation must reject it and rerun
    on the full radius), far too large, or none -- gives bit-identical
    observations and selection indices."""
    raw = generate(WaymoSpec(n_worlds=12, n_agents=64, n_points=3000, seed=21, quantize=False))
    cfg = SimConfig(init_mode="all_valid", dynamics="delta_local")
    a, b = (SimBatch.from_raw(raw, cfg, device="cuda:0") for _ in range(2))
    sel_w = cfg.obs.max_agents_obs + cfg.obs.max_road_points_obs
    sa, sb = (torch.full((a.n_controlled, sel_w), -7, dtype=torch.int32, device="cuda:0")
              for _ in range(2))
    rng = np.random.default_rng(4)
    a.reset(sel_idx=sa)
    b.reset(sel_idx=sb)
    for t in range(6):
        act = torch.from_numpy(actions_for(cfg, a.n_controlled, rng)).cuda()
        a.step(act, sel_idx=sa)
        b.step(act, sel_idx=sb)
        torch.cuda.synchronize()
        assert torch.equal(a.observations, b.observations) and torch.equal(sa, sb)
        # corrupt b's hint for its next step (columns: bound, x, y of the
        # position it was taken at, grid-relative)
        h = b._hint
        if hint == "bogus_small":
            h[:, 0] = 0.5
        elif hint == "bogus_large":
            h[:, 0] = 1e4
        else:
            h.zero_()
        b.observe(sel_idx=sb)
        torch.cuda.synchronize()
        assert torch.equal(a.observations, b.observations), f"step {t}: observations differ"
        assert torch.equal(sa, sb), f"step {t}: selections differ"
    a.close()
    b.close()
