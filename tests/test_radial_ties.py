"""Radial selection knife edges: road points in groups of eight at exactly
equal distances (dyadic offsets from a dyadic agent position) and at nearly
equal ones (non-dyadic offsets far from the origin), groups straddling the
64-slot cutoff and sitting exactly on the 50 m radius.  The kernel ranks by
float keys and sends near ties / possibly-out-of-radius keys to the exact
path (fp:214-302: ascending (distance, index), radius inclusive); selection
indices must equal the oracle's and observations stay within tolerance."""

import math

import numpy as np
import pytest

from paper_2408_01584_b200.config import ObsConfig, SimConfig
from paper_2408_01584_b200.packing import raw_from_prepared
from paper_2408_01584_b200.scenario import RoadElement, Vec2
from parity import obs_tolerance
from scenes import hold, scene, scripted_object


def _world(w, exact, boundary=False):
    rng = np.random.default_rng(100 + w)
    cx, cy = (1024.5, -2048.25) if exact else (1234.567891, -987.654321)
    pairs = [(3.0, 4.0), (30.0, 40.0), (0.0, 50.0)]     # radius 5, 50 (x2): boundary groups
    if boundary:
        # fewer than 64 points inside: the radius itself decides (50 m exactly
        # -- 14^2 + 48^2 = 50^2 -- is inside, 50 m + a few ulps / 1e-9 is out)
        pairs += [(14.0, 48.0), (0.0, 50.0 + 1e-9), (30.0, 40.0 + 4e-14), (0.0, 49.999999999)]
    n_pairs = 8 if boundary else 34
    while len(pairs) < n_pairs:
        a, b = rng.uniform(2.0, 36.0, 2)
        if exact:
            a, b = round(a * 64) / 64, round(b * 64) / 64
        pairs.append((float(a), float(b)))
    roads, k = [], 0
    for a, b in pairs:
        for sx, sy, sw in [(1, 1, 0), (1, -1, 0), (-1, 1, 0), (-1, -1, 0),
                           (1, 1, 1), (1, -1, 1), (-1, 1, 1), (-1, -1, 1)]:
            dx, dy = (b, a) if sw else (a, b)
            p = Vec2(cx + sx * dx, cy + sy * dy)
            q = Vec2(cx + sx * dx + 1e-3, cy + sy * dy)       # a second point 1 mm away
            roads.append(RoadElement(id=k, kind="road_line", geometry=[p] if boundary else [p, q]))
            k += 1
    agents = [scripted_object(0, hold(cx, cy, 0.3, 3), goal=(cx + 400, cy))]
    agents += [scripted_object(i, hold(cx + 20.0 * i, cy - 7.0 * i, 0.1 * i, 3), goal=(cx, cy + 400))
               for i in range(1, 4)]
    return scene(agents, roads, name=f"ties-{w}-{int(exact)}")


@pytest.mark.gpu
@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("boundary", [False, True])
def test_tie_groups_and_radius_boundary_match_oracle(exact, boundary):
    import torch
    from oracle.oracle import OracleBatch
    from paper_2408_01584_b200.engine import SimBatch
    raw = raw_from_prepared([_world(w, exact, boundary) for w in range(6)])
    cfg = SimConfig(init_mode="all_valid", obs=ObsConfig(mode="radial", radius=50.0))
    b = SimBatch.from_raw(raw, cfg, device="cuda:0")
    ora = OracleBatch(raw, cfg)
    sel_w = cfg.obs.max_agents_obs + cfg.obs.max_road_points_obs
    sel = torch.full((b.n_controlled, sel_w), -7, dtype=torch.int32, device="cuda:0")
    b.reset(sel_idx=sel)
    for t in range(3):
        if t:
            act = np.zeros((b.n_controlled, 2), np.float32)
            b.step(torch.as_tensor(act).cuda(), sel_idx=sel)
            ora.step(act.astype(np.float64))
        torch.cuda.synchronize()
        got = sel.cpu().numpy()
        assert np.array_equal(got, ora.sel_idx), f"step {t}: selection differs"
        o = b.observations.cpu().numpy().astype(np.float64)
        ref = ora.observations.astype(np.float32).astype(np.float64)
        err = np.abs(o - ref)
        assert (err <= obs_tolerance(ora.observations)).all(), f"step {t}: obs error {err.max()}"
    n_sel = (got[:, cfg.obs.max_agents_obs:] >= 0).sum(1)
    if boundary:    # the radius, not the cap, ends the selection of the centre agent
        assert 0 < n_sel.min() and n_sel[0] < cfg.obs.max_road_points_obs
    else:           # the tie groups straddle the 64-slot cutoff
        assert n_sel.max() == cfg.obs.max_road_points_obs
    b.close()
