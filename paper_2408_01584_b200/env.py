"""Gym-style vector environment over the B200 batch: the drop-in for the
reference's ``VecDriveEnv`` (pkg/rl/src/drivesim_rl/env.py:66-124).

One row per controlled agent across all worlds.  ``step`` runs entirely on the
device with no host synchronisation: discrete joint action indices are decoded
in the step kernel (env.py:111-116), observations are normalised in the
observation kernel (env.py:50-63, 118-121), finished worlds are auto-reset in
the step kernel with the reference's buffer semantics (rewards of a reset world
read 0, dones/infos keep the final step, env.py:95-109), and
``infos["episodes"]`` is a lazy sequence that only drains the device episode
ring when it is read.

Returned tensors live on the device; ``obs`` and ``rewards`` are the batch's
buffers (zero-copy, overwritten by the next step, like the reference's
``rewards``); ``dones`` and the info flags are fresh tensors.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import RAY_WIDTH, ROAD_SLOT_WIDTH, DEFAULT_ACCEL_BOUNDS, DEFAULT_STEER_BOUNDS, \
    SimConfig, obs_width
from .engine import SimBatch

DEFAULT_ROLLOUT_LENGTH = 92


class IndexOutOfRange(IndexError):
    pass


@dataclass
class ActionGrid:
    """Row-major bijection between joint indices and (accel, steer) pairs
    (pkg/src/drivesim/dynamics.py:143-177)."""

    accelerations: list = field(
        default_factory=lambda: list(np.linspace(*DEFAULT_ACCEL_BOUNDS, 7)))
    steerings: list = field(
        default_factory=lambda: list(np.linspace(*DEFAULT_STEER_BOUNDS, 13)))

    def __post_init__(self):
        for name in ("accelerations", "steerings"):
            v = list(getattr(self, name))
            if sorted(v) != v or len(set(v)) != len(v):
                raise ValueError(f"{name[:-1]} levels must be strictly increasing")

    @property
    def size(self) -> int:
        return len(self.accelerations) * len(self.steerings)

    def discretize(self, index: int):
        if not 0 <= index < self.size:
            raise IndexOutOfRange(f"index {index} not in [0, {self.size})")
        ai, si = divmod(index, len(self.steerings))
        return float(self.accelerations[ai]), float(self.steerings[si])

    def action_index(self, accel: float, steer: float) -> int:
        ai = min(range(len(self.accelerations)), key=lambda i: abs(self.accelerations[i] - accel))
        si = min(range(len(self.steerings)), key=lambda i: abs(self.steerings[i] - steer))
        return ai * len(self.steerings) + si


@dataclass
class EnvConfig:
    scenario_paths: list = field(default_factory=list)
    scenarios: list = field(default_factory=list)   # prepared scenario objects
    sim: SimConfig = None
    num_worlds: int = 4
    rollout_length: int = DEFAULT_ROLLOUT_LENGTH
    grid: ActionGrid = field(default_factory=ActionGrid)
    normalize_obs: bool = True
    n_workers: int = 1
    device: str = "cuda"
    raw: object = None          # optional RawWorlds batch (vectorised scenes)
    # observation buffer: "float32" (the reference's values rounded to f32) or
    # "bfloat16" rows padded to a multiple of 8 (policy-GEMM ready, zero pad)
    obs_dtype: str = "float32"

    def __post_init__(self):
        if self.rollout_length < 1:
            raise ValueError("rollout_length must be >= 1")
        if self.obs_dtype not in ("float32", "bfloat16"):
            raise ValueError(f"obs_dtype must be float32 or bfloat16, got {self.obs_dtype!r}")
        if self.sim is None:
            self.sim = SimConfig(collision_behavior="remove_agent")


def obs_scale(cfg: SimConfig) -> np.ndarray:
    """Per-feature divisors of the flat observation vector (env.py:50-63)."""
    o = cfg.obs
    pos = o.radius if o.mode == "radial" else o.max_range
    ego = np.array([cfg.v_max, 10.0, 10.0, pos, pos, pos, 1.0])
    if o.mode == "radial":
        partner = np.array([pos, pos, np.pi, cfg.v_max, 10.0, 10.0, 1.0])
        road = np.concatenate([[pos, pos, np.pi], np.ones(ROAD_SLOT_WIDTH - 3)])
        return np.concatenate([ego, np.tile(partner, o.max_agents_obs),
                               np.tile(road, o.max_road_points_obs)])
    ray = np.concatenate([[o.max_range], np.ones(RAY_WIDTH - 1)])
    return np.concatenate([ego, np.tile(ray, o.n_rays)])


class LazyEpisodes(Sequence):
    """The EpisodeInfo records of one step; drains the device ring (a host
    synchronisation) only when first read."""

    def __init__(self, batch: SimBatch, serial: int):
        self._batch, self._serial, self._items = batch, serial, None

    def _get(self):
        if self._items is None:
            self._items = self._batch.episodes_of_step(self._serial)
        return self._items

    def __len__(self):
        return len(self._get())

    def __getitem__(self, i):
        return self._get()[i]

    def __repr__(self):
        return repr(self._get())


class VecDriveEnv:
    """Vectorised per-agent environment on one GPU; auto-resets finished worlds."""

    def __init__(self, cfg: EnvConfig):
        self.cfg = cfg
        scenarios = list(cfg.scenarios)
        for path in cfg.scenario_paths:
            from .scenario import load_prepared
            with open(path) as f:
                scenarios.append(load_prepared(f.read()))
        if cfg.raw is None and not scenarios:
            raise ValueError("EnvConfig needs scenarios or scenario_paths")
        if cfg.raw is not None:
            self.scenarios = []
            self.batch = SimBatch.from_raw(cfg.raw, cfg.sim, device=cfg.device)
        else:
            self.scenarios = [scenarios[w % len(scenarios)] for w in range(cfg.num_worlds)]
            self.batch = SimBatch(self.scenarios, cfg.sim, device=cfg.device)
        self.batch.log_episodes = False   # per-step records only (env.py:103-104)
        dev = self.batch.device
        self.device = dev
        self.grid = cfg.grid
        self.n_agents = self.batch.n_controlled
        self.obs_width = obs_width(cfg.sim.obs)
        self.n_actions = self.grid.size
        if cfg.obs_dtype == "bfloat16":
            self.batch.set_obs_format(torch.bfloat16, (self.obs_width + 7) // 8 * 8)
        self._scale = (torch.tensor(obs_scale(cfg.sim), dtype=torch.float32, device=dev)
                       if cfg.normalize_obs else None)
        self._accels = torch.tensor(self.grid.accelerations, dtype=torch.float64, device=dev)
        self._steers = torch.tensor(self.grid.steerings, dtype=torch.float64, device=dev)

    # -- gym-style surface ---------------------------------------------------

    def reset(self) -> torch.Tensor:
        return self.batch.reset(obs_scale=self._scale)

    def step(self, actions):
        """actions: (n_agents,) joint indices or (n_agents, >=2) floats.
        Host joint indices are range-checked here (IndexError, as the
        reference's to_continuous); device ones by the kernel, reported by
        SimBatch.check_status at the next episode drain."""
        a = torch.as_tensor(actions)
        if a.ndim == 1 and a.device.type == "cpu" and a.numel():
            n = len(self.grid.accelerations) * len(self.grid.steerings)
            if int(a.min()) < -n or int(a.max()) >= n:
                raise IndexError(f"joint action index outside [-{n}, {n})")
        serial = self.batch._serial
        if a.ndim == 1:
            out = self.batch.step(None, action_idx=a, grid=(self._accels, self._steers),
                                  obs_scale=self._scale, auto_reset=True)
        else:
            out = self.batch.step(a, obs_scale=self._scale, auto_reset=True)
        infos = {k: v.clone() for k, v in out.info.items()}
        infos["episodes"] = LazyEpisodes(self.batch, serial)
        return out.observations, out.rewards, out.dones.clone(), infos

    def to_continuous(self, actions) -> torch.Tensor:
        a = torch.as_tensor(actions)
        if a.ndim == 2:
            return a.to(torch.float64)
        idx = a.to(torch.int64).to(self._accels.device)
        ns = len(self.grid.steerings)
        ai = torch.div(idx, ns, rounding_mode="floor")
        si = idx - ai * ns
        return torch.stack([self._accels[ai], self._steers[si]], 1)

    def close(self):
        self.batch.close()
