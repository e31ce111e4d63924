"""HostStepper (host action buffers, copies overlapped with the kernels) gives
exactly the results of SimBatch.step on the same actions: rewards, dones,
info of every step and the final observations / poses, over a full episode
with auto-reset and a depth-2 / depth-3 pipeline."""

import numpy as np
import pytest
import torch

from paper_2408_01584_b200.config import SimConfig
from paper_2408_01584_b200.engine import ActionCountMismatch, HostStepper, SimBatch
from paper_2408_01584_b200.synthetic import WaymoSpec, generate
from parity import actions_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("depth,pinned,zero_copy", [(2, True, True), (2, True, False),
                                                    (3, False, False)])
def test_host_stepper_matches_device_step(depth, pinned, zero_copy):
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent")
    raw = generate(WaymoSpec(n_worlds=6, n_agents=48, n_points=1500, seed=5))
    ref = SimBatch.from_raw(raw, cfg, device="cuda:0")
    dut = SimBatch.from_raw(raw, cfg, device="cuda:0")
    stepper = HostStepper(dut, depth=depth)
    rng = np.random.default_rng(3)
    n = ref.n_controlled
    results = []
    for t in range(100):      # > one 91-step episode: auto-reset inside
        a = torch.from_numpy(actions_for(cfg, n, rng).astype(np.float32))
        if pinned:
            a = a.pin_memory()
        out = ref.step(a.cuda(), auto_reset=True)
        want = (out.rewards.cpu().numpy(), out.dones.cpu().numpy(),
                ref._info[:, :n].cpu().numpy())
        got = stepper.step(a if pinned else a.numpy(), zero_copy=zero_copy)
        results.append((want, got))
        if len(results) >= depth:           # read each result before its slot is reused
            (w_rew, w_done, w_info), g = results.pop(0)
            g.wait()
            assert np.array_equal(g.rewards.numpy(), w_rew)
            assert np.array_equal(g.dones.numpy(), w_done)
            for i, k in enumerate(("goal", "veh_collision", "offroad")):
                assert np.array_equal(g.info[k].numpy(), w_info[i])
    stepper.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(ref.observations, dut.observations)
    for k in ("_x", "_y", "_h", "_v", "_flags"):
        assert torch.equal(getattr(ref, k), getattr(dut, k))
    ref.close()
    dut.close()


def test_host_stepper_caller_may_reuse_one_buffer():
    """The default (staged) path: the caller overwrites ONE pinned buffer with
    the next step's actions right after step() returns, without waiting."""
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent")
    raw = generate(WaymoSpec(n_worlds=4, n_agents=40, n_points=1200, seed=6))
    ref = SimBatch.from_raw(raw, cfg, device="cuda:0")
    dut = SimBatch.from_raw(raw, cfg, device="cuda:0")
    stepper = HostStepper(dut, depth=2)
    rng = np.random.default_rng(8)
    buf = torch.empty((ref.n_controlled, 2), dtype=torch.float32).pin_memory()
    for t in range(40):
        buf.copy_(torch.from_numpy(actions_for(cfg, ref.n_controlled, rng)))
        ref.step(buf.cuda(), auto_reset=True)
        stepper.step(buf)
        buf.fill_(1e3)                    # clobber it at once: must not leak into the step
    stepper.synchronize()
    torch.cuda.synchronize()
    for k in ("_x", "_y", "_h", "_v", "_flags"):
        assert torch.equal(getattr(ref, k), getattr(dut, k))
    assert torch.equal(ref.observations, dut.observations)
    ref.close()
    dut.close()


def test_host_stepper_rejects_bad_actions():
    cfg = SimConfig(init_mode="all_valid")
    raw = generate(WaymoSpec(n_worlds=2, n_agents=8, n_points=200, seed=1))
    b = SimBatch.from_raw(raw, cfg, device="cuda:0")
    s = HostStepper(b)
    with pytest.raises(ActionCountMismatch):
        s.step(np.zeros((b.n_controlled + 1, 2), np.float32))
    with pytest.raises(ValueError):
        s.step(torch.zeros((b.n_controlled, 2), device="cuda:0"))
    with pytest.raises(ValueError):                  # zero_copy needs pinned float32
        s.step(torch.zeros((b.n_controlled, 2)), zero_copy=True)
    b.close()
