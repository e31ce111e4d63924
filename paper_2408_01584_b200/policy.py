"""In-loop policy for the RL rollout configuration (BASELINE config 5).

The reference trainer's ActorCritic (pkg/rl/src/drivesim_rl/ippo.py:48-66):
a two-layer tanh MLP trunk with policy and value heads.  In the B200 loop it
runs on the same device as the simulator on the zero-copy observation buffer
(bf16 autocast -> cuBLAS tensor-core GEMMs) and samples the joint action
indices that the step kernel decodes; nothing crosses to the host.
"""

from __future__ import annotations

import torch
from torch import nn


class ActorCritic(nn.Module):
    """ippo.py:48-66.  ``pad_to`` > 1 pads the input width and the policy
    head's output count to multiples of ``pad_to`` (zero-padded observation
    columns, extra logits sliced off): the same function with 16-B aligned
    GEMM operands, so a bf16 policy gets the tensor-core GEMM kernels."""

    def __init__(self, obs_width: int, n_actions: int, hidden=(256, 256), pad_to: int = 1):
        super().__init__()
        rnd = lambda v: (v + pad_to - 1) // pad_to * pad_to
        self.obs_width, self.n_actions = obs_width, n_actions
        self.in_features = rnd(obs_width)
        layers, last = [], self.in_features
        for h in hidden:
            layers += [nn.Linear(last, h), nn.Tanh()]
            last = h
        self.trunk = nn.Sequential(*layers)
        self.policy = nn.Linear(last, rnd(n_actions))
        self.value = nn.Linear(last, 1)
        nn.init.orthogonal_(self.policy.weight, gain=0.01)
        nn.init.zeros_(self.policy.bias)

    def _input(self, obs):
        if obs.shape[1] == self.in_features:
            return obs
        # a [n, obs_width] view of a zero-padded [n, in_features] buffer (the
        # env's bf16 observation buffer): use the padded rows, no copy
        if (obs.stride(1) == 1 and obs.stride(0) == self.in_features
                and obs.storage_offset() + obs.shape[0] * self.in_features
                <= obs.untyped_storage().nbytes() // obs.element_size()):
            return obs.as_strided((obs.shape[0], self.in_features), (self.in_features, 1))
        return nn.functional.pad(obs, (0, self.in_features - obs.shape[1]))

    def forward(self, obs):
        z = self.trunk(self._input(obs))
        return self.policy(z)[:, :self.n_actions], self.value(z).squeeze(-1)


def sample_actions(logits: torch.Tensor, generator: torch.Generator | None = None) -> torch.Tensor:
    """Categorical sample per row (Gumbel-max: argmax(logits - log(-log u)))."""
    u = torch.rand(logits.shape, device=logits.device, dtype=torch.float32, generator=generator)
    g = -torch.log(-torch.log(u.clamp_min_(1e-20)))
    return torch.argmax(logits.float() + g, dim=-1).to(torch.int32)
