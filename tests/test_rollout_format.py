"""Device-rollout formats (BASELINE config 5): bf16 / padded
observation buffers, the padded ActorCritic, and the in-loop categorical
sampler.  The float32 path is the parity-checked one (test_gpu_parity.py);
these tests pin the other formats to it bit for bit."""

import numpy as np
import pytest
import torch

from paper_2408_01584_b200.config import ObsConfig, SimConfig
from paper_2408_01584_b200.policy import ActorCritic
from paper_2408_01584_b200.synthetic import WaymoSpec, generate


def test_padded_actor_critic_is_the_same_function():
    torch.manual_seed(0)
    ref = ActorCritic(823, 91)
    pad = ActorCritic(823, 91, pad_to=8)
    assert pad.in_features == 824 and pad.policy.out_features == 96
    with torch.no_grad():
        pad.trunk[0].weight.zero_()
        pad.trunk[0].weight[:, :823] = ref.trunk[0].weight
        pad.trunk[0].bias.copy_(ref.trunk[0].bias)
        pad.trunk[2].load_state_dict(ref.trunk[2].state_dict())
        pad.policy.weight.zero_()
        pad.policy.weight[:91] = ref.policy.weight
        pad.policy.bias.zero_()
        pad.policy.bias[:91] = ref.policy.bias
        pad.value.load_state_dict(ref.value.state_dict())
    obs = torch.randn(64, 823)
    buf = torch.zeros(64, 824)
    buf[:, :823] = obs
    view = buf[:, :823]                      # the env's padded-buffer view
    with torch.no_grad():
        l0, v0 = ref(obs)
        for x in (obs, view, buf):
            l1, v1 = pad(x)
            assert l1.shape == (64, 91)
            torch.testing.assert_close(l1, l0, rtol=1e-5, atol=1e-6)
            torch.testing.assert_close(v1, v0, rtol=1e-5, atol=1e-6)


def _batch(mode, **kw):
    from paper_2408_01584_b200.engine import SimBatch
    raw = generate(WaymoSpec(n_worlds=6, n_agents=24, n_points=600, seed=5, num_steps=30))
    obs = ObsConfig(mode=mode, max_agents_obs=8, max_road_points_obs=16, n_rays=12, **kw)
    sim = SimConfig(collision_behavior="remove_agent", obs=obs, init_mode="all_valid")
    return SimBatch.from_raw(raw, sim, device="cuda:0"), sim


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["radial", "lidar"])
@pytest.mark.parametrize("scaled", [True, False])
def test_bf16_and_padded_obs_match_float32(mode, scaled):
    # unscaled float32 radial rows leave through the bulk (TMA) row store,
    # scaled ones through the per-element path: both at every row phase
    from paper_2408_01584_b200.engine import random_actions
    from paper_2408_01584_b200.env import obs_scale
    ref, sim = _batch(mode)
    b16, _ = _batch(mode)
    f32p, _ = _batch(mode)
    W = ref.width
    pad8 = (W + 7) // 8 * 8
    b16.set_obs_format(torch.bfloat16, pad8)
    f32p.set_obs_format(torch.float32, W + 5)
    scale = torch.tensor(obs_scale(sim), dtype=torch.float32, device="cuda:0") if scaled else None
    for b in (ref, b16, f32p):
        b.reset(obs_scale=scale)
    for t in range(25):
        act = random_actions(ref.n_controlled, sim, 3, t, "cuda:0")
        outs = [b.step(act, obs_scale=scale, auto_reset=True) for b in (ref, b16, f32p)]
        o32 = outs[0].observations
        assert torch.equal(outs[2].observations, o32)
        assert torch.equal(outs[1].observations, o32.to(torch.bfloat16))
        assert outs[1].observations.stride(0) == pad8
        assert not b16._obs_buf[:, W:].any() and not f32p._obs_buf[:, W:].any()
        for k in (1, 2):
            assert torch.equal(outs[k].rewards, outs[0].rewards)
            assert torch.equal(outs[k].dones, outs[0].dones)


@pytest.mark.gpu
def test_env_bf16_observations():
    from paper_2408_01584_b200.env import EnvConfig, VecDriveEnv
    raw = generate(WaymoSpec(n_worlds=3, n_agents=16, n_points=400, seed=2, num_steps=12))
    sim = SimConfig(collision_behavior="remove_agent", init_mode="all_valid",
                    obs=ObsConfig(max_agents_obs=8, max_road_points_obs=16))
    e32 = VecDriveEnv(EnvConfig(raw=raw, sim=sim, device="cuda:0"))
    e16 = VecDriveEnv(EnvConfig(raw=raw, sim=sim, device="cuda:0", obs_dtype="bfloat16"))
    assert torch.equal(e16.reset(), e32.reset().to(torch.bfloat16))
    gen = np.random.default_rng(0)
    for _ in range(15):
        a = torch.as_tensor(gen.integers(0, 91, e32.n_agents), device="cuda:0")
        o32, r32, d32, _ = e32.step(a)
        o16, r16, d16, _ = e16.step(a)
        assert o16.dtype == torch.bfloat16 and o16.shape == o32.shape
        assert torch.equal(o16, o32.to(torch.bfloat16))
        assert torch.equal(r16, r32) and torch.equal(d16, d32)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_sampler_deterministic_and_distributed(dtype):
    from paper_2408_01584_b200.engine import sample_categorical
    rows, n = 4096, 91
    gen = torch.Generator().manual_seed(0)
    logits = (torch.randn(rows, 8, generator=gen) * 1.5).repeat(1, 12)[:, :n]
    logits = logits.to(dtype).cuda()
    padded = torch.full((rows, 96), 1e4, dtype=dtype, device="cuda")   # ld 96, pad ignored
    padded[:, :n] = logits
    a = sample_categorical(logits, seed=7, counter=3)
    b = sample_categorical(logits, seed=7, counter=3)
    c = sample_categorical(padded[:, :n], seed=7, counter=3)
    d = sample_categorical(logits, seed=7, counter=4)
    assert torch.equal(a, b) and torch.equal(a, c)
    assert (a != d).float().mean() > 0.3
    assert int(a.min()) >= 0 and int(a.max()) < n
    # empirical frequencies over many counters against softmax, one shared row
    row = logits[:1].expand(20000, n).contiguous()
    counts = torch.zeros(n, dtype=torch.float64)
    for k in range(10):
        s = sample_categorical(row, seed=11, counter=100 + k).cpu()
        counts += torch.bincount(s.to(torch.int64), minlength=n).double()
    p = torch.softmax(row[0].float().cpu().double(), 0)
    expect = p * counts.sum()
    chi2 = float(((counts - expect) ** 2 / expect.clamp_min(1e-9))[expect > 5].sum())
    dof = int((expect > 5).sum()) - 1
    assert chi2 < dof + 6 * (2 * dof) ** 0.5


@pytest.mark.gpu
def test_gumbel_noise_at_the_hash_extremes():
    """The sampler's noise is finite and accurate for every hash value,
    including the maximum (u = 1 - 2^-24, where a naive float u would round
    to 1 and -log(-log u) to +inf): against float64 -log(-log u)."""
    import ctypes as C
    from paper_2408_01584_b200 import _native as N
    rng = np.random.default_rng(0)
    bits = np.concatenate([np.array([0, 0x1FF, 0x200, 0xFFFFFFFF, 0xFFFFFE00, 0xFFFFFDFF,
                                     0x80000000, 0x7FFFFFFF], np.uint32),
                           rng.integers(0, 2**32, 4096, dtype=np.uint64).astype(np.uint32)])
    dev_bits = torch.from_numpy(bits.view(np.int32)).cuda()
    out = torch.empty(len(bits), dtype=torch.float32, device="cuda")
    N.check(N.lib().ds_gumbel_noise(C.c_void_p(dev_bits.data_ptr()), len(bits),
                                    C.c_void_p(out.data_ptr()), None), "ds_gumbel_noise")
    got = out.cpu().numpy().astype(np.float64)
    m = (bits >> 9).astype(np.float64)
    u = (2 * m + 1) / 2.0**24
    ref = -np.log(-np.log1p(-(1 - u)))
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 4e-6 * np.maximum(1.0, np.abs(ref)).max()
    assert got[3] == got.max() and got[3] > 16.0          # u = 1 - 2^-24: the largest noise
