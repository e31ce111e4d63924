"""The C oracle and the packer, pinned to the real reference through the
golden fixtures: bit-exact observations (SHA-256 of every step's float64
buffer), rewards, dones, info flags, poses and episode records over full
91-step episodes, plus the World.__init__ tables."""

import numpy as np
import pytest

from golden_util import NAMES, load, sha
from oracle.oracle import OracleBatch
from oracle.tables import build_tables
from paper_2408_01584_b200.packing import pack


@pytest.mark.parametrize("builder", ["product_packer", "oracle_tables"])
@pytest.mark.parametrize("name", NAMES)
def test_tables_match_reference_world_tables(name, builder):
    """Both table builders -- the product packer (vectorised) and the
    oracle's own restatement (oracle/tables.py) -- reproduce the reference's
    World.__init__ tables bit for bit."""
    z, raw, cfg = load(name)
    pw = pack(raw, cfg) if builder == "product_packer" else build_tables(raw, cfg)
    for w in range(pw.n_worlds):
        A = int(pw.a_off[w + 1] - pw.a_off[w])
        T = int(pw.num_steps[w])
        sl = slice(int(pw.r_off[w]), int(pw.r_off[w]) + A * T)
        assert np.array_equal(pw.rep_x[sl].reshape(T, A).T, z[f"tab{w}_replay_pos"][:, :, 0])
        assert np.array_equal(pw.rep_y[sl].reshape(T, A).T, z[f"tab{w}_replay_pos"][:, :, 1])
        assert np.array_equal(pw.rep_h[sl].reshape(T, A).T, z[f"tab{w}_replay_heading"])
        assert np.array_equal(pw.rep_v[sl].reshape(T, A).T, z[f"tab{w}_replay_speed"])
        assert np.array_equal(pw.rep_present[sl].reshape(T, A).T.astype(bool),
                              z[f"tab{w}_present_log"])
        assert np.array_equal(pw.controlled_ids(w), z[f"tab{w}_controlled_ids"])
        p0, p1 = int(pw.p_off[w]), int(pw.p_off[w + 1])
        assert np.array_equal(pw.pt_h[p0:p1], z[f"tab{w}_road_pt_heading"])
        a0, a1 = int(pw.a_off[w]), int(pw.a_off[w + 1])
        assert np.array_equal(pw.circumradius[a0:a1], z[f"tab{w}_circumradius"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_bit_exact_vs_reference(name):
    z, raw, cfg = load(name)
    OracleBatch.lidar_ties()                 # reset the tie counter
    ora = OracleBatch(raw, cfg)
    assert sha(ora.observations) == z["obs_sha256"][0]
    steps = z["actions"].shape[0]
    for t in range(1, steps + 1):
        obs, rew, done, info = ora.step(z["actions"][t - 1].astype(np.float64))
        assert np.array_equal(rew, z["rewards"][t - 1]), t
        assert np.array_equal(done, z["dones"][t - 1]), t
        for k, key in enumerate(("goal", "veh_collision", "offroad")):
            assert np.array_equal(info[key], z["info"][t - 1, k]), (t, key)
        assert sha(obs) == z["obs_sha256"][t], f"step {t}: observations differ"
        pos = np.stack([ora.x[:ora.pw.n_agents], ora.y[:ora.pw.n_agents],
                        ora.heading[:ora.pw.n_agents], ora.speed[:ora.pw.n_agents]])
        assert np.array_equal(pos, z["poses"][t - 1]), f"step {t}: poses differ"
    eps = np.array(ora.episode_infos, np.int64).reshape(-1, 5)
    assert np.array_equal(eps, z["episodes"])
    # no ray of these episodes met an edge / non-edge exact tie, the one
    # LiDAR case where the reference's answer follows its BVH order
    assert OracleBatch.lidar_ties() == 0
