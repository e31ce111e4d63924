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
    def __init__(self, obs_width: int, n_actions: int, hidden=(256, 256)):
        super().__init__()
        layers, last = [], obs_width
        for h in hidden:
            layers += [nn.Linear(last, h), nn.Tanh()]
            last = h
        self.trunk = nn.Sequential(*layers)
        self.policy = nn.Linear(last, n_actions)
        self.value = nn.Linear(last, 1)
        nn.init.orthogonal_(self.policy.weight, gain=0.01)
        nn.init.zeros_(self.policy.bias)

    def forward(self, obs):
        z = self.trunk(obs)
        return self.policy(z), self.value(z).squeeze(-1)


def sample_actions(logits: torch.Tensor, generator: torch.Generator | None = None) -> torch.Tensor:
    """Categorical sample per row (Gumbel-max: argmax(logits - log(-log u)))."""
    u = torch.rand(logits.shape, device=logits.device, dtype=torch.float32, generator=generator)
    g = -torch.log(-torch.log(u.clamp_min_(1e-20)))
    return torch.argmax(logits.float() + g, dim=-1).to(torch.int32)
