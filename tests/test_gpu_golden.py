"""The CUDA path against the real reference's golden trajectories (made by
tests/golden/make_golden.py): flags bit-exact at every step, float32
observations within 2 ulp + 1e-6 of the reference's float64 at every stored
step, FP64 poses within 1e-9 m / 1e-12 rad at every step."""

import numpy as np
import pytest
import torch

from golden_util import NAMES, load
from parity import ANG_TOL, POS_TOL, obs_tolerance, wrap_diff
from paper_2408_01584_b200.engine import SimBatch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference_golden(name):
    z, raw, cfg = load(name)
    if cfg.obs.mode != "radial":
        from paper_2408_01584_b200 import _native
        if not _native.lidar_supported():
            pytest.skip("LiDAR kernel not built")
    batch = SimBatch.from_raw(raw, cfg, device="cuda:0")

    def check_obs(t):
        if f"obs_{t}" not in z:
            return
        ref = z[f"obs_{t}"]
        got = batch.observations.cpu().numpy().astype(np.float64)
        err = np.abs(got - ref.astype(np.float32).astype(np.float64))
        assert (err <= obs_tolerance(ref)).all(), f"step {t}: max err {err.max()}"

    check_obs(0)
    steps = z["actions"].shape[0]
    nA = batch.packed.n_agents
    for t in range(1, steps + 1):
        out = batch.step(torch.from_numpy(z["actions"][t - 1]).cuda())
        assert np.array_equal(out.rewards.cpu().numpy(), z["rewards"][t - 1].astype(np.float32))
        assert np.array_equal(out.dones.cpu().numpy(), z["dones"][t - 1])
        info = batch._info[:, :batch.n_controlled].cpu().numpy()
        assert np.array_equal(info, z["info"][t - 1]), f"step {t}"
        check_obs(t)
        pose = z["poses"][t - 1]
        assert np.abs(batch._x.cpu().numpy()[:nA] - pose[0]).max() <= POS_TOL, f"step {t}"
        assert np.abs(batch._y.cpu().numpy()[:nA] - pose[1]).max() <= POS_TOL, f"step {t}"
        assert wrap_diff(batch._h.cpu().numpy()[:nA], pose[2]).max() <= ANG_TOL, f"step {t}"
        assert np.abs(batch._v.cpu().numpy()[:nA] - pose[3]).max() <= POS_TOL, f"step {t}"
    eps = np.array([(e.world_id, e.n_controlled, e.n_goal, e.n_veh_collision, e.n_offroad)
                    for e in batch.episode_infos], np.int64).reshape(-1, 5)
    assert np.array_equal(eps, z["episodes"])
    batch.close()
